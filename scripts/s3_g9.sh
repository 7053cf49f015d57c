L=$PWD/paper_2104_12282_b200/lib
for v in libtomo_dc libtomo_dc16; do
  echo "== $v"; TOMO_LIB_PATH=$L/$v.so timeout 100 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
done
bash scripts/ab_time.sh cfg3 400 libtomo libtomo_dc libtomo_dc16
