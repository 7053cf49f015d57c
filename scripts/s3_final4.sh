# final round-1 session-3 evidence on the committed kernel: launch list + ncu of both kernels
O=gpurun_out
export TOMO_NO_GRAPH=1
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/s3k_plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file $O/s3k_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/s3k_ncu_ll.log 2>&1
python scripts/prof_step.py cfg3 24 > $O/s3k_plain2.log 2>&1 && python scripts/time_apply.py cfg3 > $O/s3k_plain3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_op" -s 10 -c 1 -o $O/s3k_pcg python scripts/prof_step.py cfg3 24 > $O/s3k_ncu3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_op" -s 5 -c 1 -o $O/s3k_apply python scripts/time_apply.py cfg3 > $O/s3k_ncu4.log 2>&1
ls $O | grep s3k
