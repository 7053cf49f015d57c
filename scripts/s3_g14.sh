timeout 900 python scripts/sweep_cfg4.py gpurun_out/s3_sweep_full.json > gpurun_out/s3_sweep_full.log 2>&1; tail -3 gpurun_out/s3_sweep_full.log
