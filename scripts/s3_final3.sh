O=gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/s3h_smoke.log 2>&1; tail -2 $O/s3h_smoke.log
timeout 900 python bench.py > $O/s3h_bench.log 2>&1; tail -1 $O/s3h_bench.log | cut -c1-150
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > $O/s3h_ref.log 2>&1; tail -1 $O/s3h_ref.log | cut -c1-150
