#!/bin/bash
# A/B timing of prebuilt library variants (scripts/build_variants.py) on the GPU box:
#   bash scripts/ab.sh TAG lib1 lib2 ...   (lib = name under paper_2104_12282_b200/lib, no .so)
# per variant: parity subset, PCG launch time at cfg3 (time_kernel.py), K_hat u (time_apply.py);
# the variants alternate twice so that clock drift shows up.
TAG=$1; shift
O=gpurun_out; mkdir -p $O
L=paper_2104_12282_b200/lib
for v in "$@"; do
  TOMO_LIB_PATH=$PWD/$L/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "not cfg3" \
    > $O/${TAG}_${v}_tests.log 2>&1; echo "$v tests: $(tail -1 $O/${TAG}_${v}_tests.log)"
done
for rep in 1 2; do
  for v in "$@"; do
    TOMO_LIB_PATH=$PWD/$L/$v.so timeout 300 python scripts/time_kernel.py cfg3 400 2>&1 | tail -1
    TOMO_LIB_PATH=$PWD/$L/$v.so timeout 300 python scripts/time_apply.py cfg3 4.4 2>&1 | tail -2
  done
done
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv
