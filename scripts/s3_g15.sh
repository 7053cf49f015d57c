bash scripts/ab_time.sh cfg3 400 libtomo libtomo_c1 libtomo_c3
for v in libtomo_c1 libtomo_c3; do TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1; done
