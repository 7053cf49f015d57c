for r in 1; do
timeout 120 python scripts/time_kernel.py cfg4e 200
TOMO_SCHED=sync timeout 120 python scripts/time_kernel.py cfg4e 200
TOMO_SCHED=sync TOMO_ZCHUNKS=2 timeout 120 python scripts/time_kernel.py cfg4e 200
TOMO_SCHED=sync TOMO_ZCHUNKS=3 timeout 120 python scripts/time_kernel.py cfg4e 200
TOMO_SCHED=sync TOMO_ZCHUNKS=4 timeout 120 python scripts/time_kernel.py cfg4e 200
TOMO_SCHED=sync TOMO_ZCHUNKS=3 timeout 120 python scripts/time_kernel.py cfg3 300
TOMO_SCHED=sync TOMO_ZCHUNKS=4 timeout 120 python scripts/time_kernel.py cfg3 300
done
