for r in 1 2; do
TOMO_NO_REV=1 timeout 120 python scripts/time_kernel.py cfg3 400
timeout 120 python scripts/time_kernel.py cfg3 400
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
