bash scripts/ab_time.sh cfg3 400 libtomo libtomo_rl0 libtomo_rl2 libtomo_rl8 libtomo_rl10
for v in libtomo libtomo_rl0 libtomo_rl10; do TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/$v.so timeout 120 python scripts/time_apply.py cfg3; done
