#!/bin/bash
# A/B of K_hat u build variants: operator parity (all grids, edges, mg), then time_apply twice alternating
#   bash scripts/explore/apply_ab.sh TAG lib1 lib2 ...
TAG=$1; shift
O=gpurun_out; mkdir -p $O
L=paper_2104_12282_b200/lib
for v in "$@"; do
  TOMO_LIB_PATH=$PWD/$L/$v.so timeout 600 python -m pytest tests -m gpu -q -k "apply or operator or mg or edges or abi or twoscale" > $O/${TAG}_${v}_tests.log 2>&1
  echo "$v tests: $(tail -1 $O/${TAG}_${v}_tests.log)"
done
for rep in 1 2; do
  for v in "$@"; do
    TOMO_LIB_PATH=$PWD/$L/$v.so timeout 300 python scripts/time_apply.py cfg3 4.3 4.4 2>&1 | tail -3
  done
done | tee $O/${TAG}_apply_ab.log
