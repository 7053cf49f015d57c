for v in libtomo libtomo_ag libtomo_m3 libtomo_m3g; do TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/$v.so timeout 120 python scripts/time_apply.py cfg3 4.4; done
bash scripts/ab_time.sh cfg3 400 libtomo libtomo_pg
timeout 300 python -m pytest tests -m gpu -q -x -k "apply or op or mg" 2>&1 | tail -2
