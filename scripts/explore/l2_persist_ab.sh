#!/bin/bash
# A/B: E and D^-1 (1) / and u (2) as a persisting L2 window (TOMO_L2_PERSIST) on the stream and the
# graph's PCG kernel nodes; graph mode (default) and host-batched launches (TOMO_NO_GRAPH=1)
for rep in 1 2; do
  for v in 0 1; do
    if [ $v = 0 ]; then unset TOMO_L2_PERSIST; else export TOMO_L2_PERSIST=$v; fi
    echo "== persist $v"; timeout 300 python scripts/time_iter.py cfg3 400 2>&1 | tail -1
    TOMO_NO_GRAPH=1 timeout 300 python scripts/time_iter.py cfg3 400 2>&1 | tail -1
  done
done | tee gpurun_out/${1:-x}_l2_persist_ab.log
