bash scripts/ab_time.sh cfg3 400 libtomo_ref libtomo libtomo_cp libtomo_t0 libtomo_pp
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
