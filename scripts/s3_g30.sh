for v in libtomo libtomo_b16 libtomo_b12; do TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/$v.so timeout 120 python scripts/time_apply.py cfg3 4.3 4.4; done
