export TOMO_NO_GRAPH=1
export TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/libtomo_pp.so
python scripts/prof_step.py cfg3 24 > gpurun_out/s3i_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:"k_op" -s 10 -c 1 -o gpurun_out/s3i_pp python scripts/prof_step.py cfg3 24 > gpurun_out/s3i_ncu.log 2>&1
tail -1 gpurun_out/s3i_ncu.log
