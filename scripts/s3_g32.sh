for v in libtomo_ref libtomo; do TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/$v.so timeout 120 python scripts/time_apply.py cfg3 4.3 4.4; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
