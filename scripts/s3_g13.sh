for r in 1 2; do
timeout 120 python scripts/time_kernel.py cfg3 400
TOMO_SCHED=balanced timeout 120 python scripts/time_kernel.py cfg3 400
done
