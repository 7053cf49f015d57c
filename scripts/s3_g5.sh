TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/libtomo_ag.so timeout 120 python scripts/time_apply.py cfg3 4.4
export TOMO_NO_GRAPH=1
python scripts/prof_step.py cfg3 12 > gpurun_out/s3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_op" -s 4 -c 1 -o gpurun_out/s3_pcg2 python scripts/prof_step.py cfg3 12 > gpurun_out/s3_ncu.log 2>&1
tail -1 gpurun_out/s3_ncu.log
