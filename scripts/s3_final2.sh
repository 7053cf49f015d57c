# round-1 session-3 final measurement (after the face-transform changes)
O=gpurun_out
timeout 900 python bench.py > $O/s3g_bench.log 2>&1; tail -1 $O/s3g_bench.log | cut -c1-200
timeout 900 python scripts/sweep_cfg4.py $O/s3g_sweep.json > $O/s3g_sweep.log 2>&1; tail -1 $O/s3g_sweep.log | cut -c1-100
export TOMO_NO_GRAPH=1
python scripts/prof_step.py cfg3 24 > $O/s3g_plain2.log 2>&1 && python scripts/time_apply.py cfg3 > $O/s3g_plain3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_op" -s 10 -c 1 -o $O/s3g_pcg python scripts/prof_step.py cfg3 24 > $O/s3g_ncu3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_op" -s 5 -c 1 -o $O/s3g_apply python scripts/time_apply.py cfg3 > $O/s3g_ncu4.log 2>&1
ls $O | grep s3g
