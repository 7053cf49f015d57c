#!/bin/bash
# One GPU iteration: parity tests, a short bench, then an ncu capture of K_A and K_B.
# usage: scripts/gpu_cycle.sh TAG [skip_tests]
TAG=${1:-cycle}
O=gpurun_out
if [ "$2" != "skip_tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $O/${TAG}_tests.log 2>&1
  tail -3 $O/${TAG}_tests.log
fi
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/${TAG}_bench.log 2>&1
tail -1 $O/${TAG}_bench.log | cut -c1-200
python scripts/prof_step.py cfg3 12 > $O/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_op|k_pcg_b" -s 4 -c 2 -o $O/${TAG}_prof python scripts/prof_step.py cfg3 12 > $O/${TAG}_ncu.log 2>&1
echo cycle-done
