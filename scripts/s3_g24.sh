bash scripts/ab_time.sh cfg3 400 libtomo_ref libtomo
for c in cfg4d cfg4e cfg2; do for v in libtomo_ref libtomo; do TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/$v.so timeout 120 python scripts/time_kernel.py $c 300; done; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
