#!/bin/bash
# A/B of the TMA tensor maps' L2 promotion (TOMO_TMA_L2PROMO = 0 none | 1 64 B | 2 128 B | 3 256 B):
# PCG iteration (scripts/time_iter.py) and K_hat u (scripts/time_apply.py) at cfg3, twice alternating.
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
  for v in 2 3 0 1; do
    echo "== promo $v"
    TOMO_TMA_L2PROMO=$v timeout 300 python scripts/time_iter.py cfg3 400 2>&1 | tail -1
    TOMO_TMA_L2PROMO=$v timeout 300 python scripts/time_apply.py cfg3 2>&1 | tail -1
  done
done | tee $O/${1:-x}_tma_promo_ab.log
