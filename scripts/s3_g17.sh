for c in cfg3 cfg4d cfg4e cfg2; do timeout 120 python scripts/time_kernel.py $c 300; done
TOMO_ZCHUNKS=3 timeout 120 python scripts/time_kernel.py cfg4e 300
timeout 200 python scripts/time_apply.py cfg3 4.3 4.4
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
