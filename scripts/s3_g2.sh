L=paper_2104_12282_b200/lib
for v in libtomo libtomo_a3 libtomo_a4 libtomo_a7; do TOMO_LIB_PATH=$PWD/$L/$v.so timeout 120 python scripts/time_apply.py cfg3 4.3 4.4; done
timeout 200 python -m pytest tests -m gpu -q -x -k "apply or op" 2>&1 | tail -2
export TOMO_NO_GRAPH=1
python scripts/prof_step.py cfg3 12 > gpurun_out/s3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_op" -s 4 -c 1 -o gpurun_out/s3_pcg python scripts/prof_step.py cfg3 12 > gpurun_out/s3_ncu.log 2>&1
tail -2 gpurun_out/s3_ncu.log
