O=gpurun_out; L=paper_2104_12282_b200/lib
for v in sens_old sens_new sens_old4 sens_new4; do
  TOMO_LIB_PATH=$PWD/$L/$v.so timeout 300 python -m pytest tests -m gpu -q -x -k "sens" > $O/sab_${v}_tests.log 2>&1; echo "$v $(tail -1 $O/sab_${v}_tests.log)"
done
for rep in 1 2; do for v in sens_old sens_new sens_old4 sens_new4; do
  echo "$v $(TOMO_LIB_PATH=$PWD/$L/$v.so timeout 300 python scripts/time_sens.py cfg3 4.4 4.3 2>&1 | tr '\n' ' ')"
done; done
