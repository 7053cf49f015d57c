# round-1 session-3 measurement: bench line, full-step launch list, ncu of the PCG and K_hat u kernels
O=gpurun_out
timeout 900 python bench.py > $O/s3_bench.log 2>&1; tail -1 $O/s3_bench.log
export TOMO_NO_GRAPH=1
timeout 300 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/s3_plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file $O/s3_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/s3_ncu_ll.log 2>&1
python scripts/prof_step.py cfg3 24 > $O/s3_plain2.log 2>&1 && python scripts/time_apply.py cfg3 > $O/s3_plain3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_op" -s 10 -c 1 -o $O/s3_pcg3 python scripts/prof_step.py cfg3 24 > $O/s3_ncu3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_op" -s 5 -c 1 -o $O/s3_apply python scripts/time_apply.py cfg3 > $O/s3_ncu4.log 2>&1
ls $O
