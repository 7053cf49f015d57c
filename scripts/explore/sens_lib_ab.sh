#!/bin/bash
# k_sens launch durations (ncu) in tomo_evaluate for library variants; sens/evaluate parity first
#   bash scripts/explore/sens_lib_ab.sh TAG lib1 lib2 ...
TAG=$1; shift
O=gpurun_out; mkdir -p $O
L=paper_2104_12282_b200/lib
for v in "$@"; do
  export TOMO_LIB_PATH=$PWD/$L/$v.so
  timeout 600 python -m pytest tests -m gpu -q -k "sens or cfg0 or cfg2 or edges" > $O/${TAG}_${v}_tests.log 2>&1
  echo "$v tests: $(tail -1 $O/${TAG}_${v}_tests.log)"
  python scripts/explore/sens_eval.py cfg3 4.3 4.4 | tail -3
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sens --csv --log-file $O/${TAG}_sens_$v.csv \
    python scripts/explore/sens_eval.py cfg3 4.3 4.4 > /dev/null 2>&1
  echo "== $v"; grep k_sens $O/${TAG}_sens_$v.csv | awk -F'","' '{print $(NF)}' | tr -d '"' | paste -sd' '
  TOMO_LIB_PATH=$PWD/$L/$v.so python scripts/time_sens.py cfg3 4.4
done
