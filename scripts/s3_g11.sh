timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
bash scripts/ab_time.sh cfg3 400 libtomo_p0 libtomo
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
