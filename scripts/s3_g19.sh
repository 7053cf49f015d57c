L=$PWD/paper_2104_12282_b200/lib
for v in libtomo_da3 libtomo_da4; do TOMO_LIB_PATH=$L/$v.so timeout 120 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1; done
for v in libtomo libtomo_da3 libtomo_da4; do TOMO_LIB_PATH=$L/$v.so timeout 120 python scripts/time_apply.py cfg3 4.3 4.4; done
