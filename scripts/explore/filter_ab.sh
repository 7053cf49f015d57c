#!/bin/bash
# A/B of tiled-filter build variants (scripts/build_variants.py): filter parity tests, then
# scripts/time_filter.py at cfg3 (93 taps), rmin 1.5 / 2.0 grids, twice alternating.
#   bash scripts/explore/filter_ab.sh TAG lib1 lib2 ...
TAG=$1; shift
O=gpurun_out; mkdir -p $O
L=paper_2104_12282_b200/lib
for v in "$@"; do
  TOMO_LIB_PATH=$PWD/$L/$v.so timeout 600 python -m pytest tests -m gpu -q -k "filter" > $O/${TAG}_${v}_tests.log 2>&1
  echo "$v tests: $(tail -1 $O/${TAG}_${v}_tests.log)"
done
for rep in 1 2; do
  for v in "$@"; do
    echo "== $v"
    TOMO_LIB_PATH=$PWD/$L/$v.so timeout 300 python scripts/time_filter.py 224 112 56 3.0 96 32 32 2.0 48 24 24 1.5 2>&1 | cut -c1-400 | tail -6
  done
done | tee $O/${TAG}_filter_ab.log
