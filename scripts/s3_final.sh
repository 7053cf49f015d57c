# round-1 session-3 final measurement: GPU tests, bench line, full-step launch list, cfg4 sweep
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/s3f_tests.log 2>&1; tail -2 $O/s3f_tests.log
timeout 900 python bench.py > $O/s3f_bench.log 2>&1; tail -1 $O/s3f_bench.log | cut -c1-300
export TOMO_NO_GRAPH=1
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/s3f_plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file $O/s3f_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/s3f_ncu_ll.log 2>&1
unset TOMO_NO_GRAPH
timeout 900 python scripts/sweep_cfg4.py $O/s3f_sweep.json > $O/s3f_sweep.log 2>&1; tail -1 $O/s3f_sweep.log | cut -c1-200
