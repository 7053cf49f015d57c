bash scripts/ab_time.sh cfg3 400 libtomo_ref libtomo
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
