for r in 1 2; do
timeout 120 python scripts/time_kernel.py cfg3 400
TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/libtomo_su.so timeout 120 python scripts/time_kernel.py cfg3 400
TOMO_EXP_SKIPU=1 TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/libtomo_su.so timeout 120 python scripts/time_kernel.py cfg3 400
done
