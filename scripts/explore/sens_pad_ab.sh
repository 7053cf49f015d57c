#!/bin/bash
# k_sens launch durations (ncu, cold-cache) in tomo_evaluate: padded row-SoA u vs dense u + mask
O=gpurun_out; mkdir -p $O
for m in pad dense; do
  if [ $m = dense ]; then export TOMO_SENS_DENSE=1; else unset TOMO_SENS_DENSE; fi
  python scripts/explore/sens_eval.py cfg3 4.3 4.4 | tail -3
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sens --csv --log-file $O/${1:-x}_sens_$m.csv \
    python scripts/explore/sens_eval.py cfg3 4.3 4.4 > /dev/null 2>&1
  echo "== $m"; grep k_sens $O/${1:-x}_sens_$m.csv | awk -F'","' '{print $(NF)}' | tr -d '"' | paste -sd' '
done
