timeout 600 python scripts/time_loop_cfg3.py gpurun_out/s3_loop_cfg3.json > gpurun_out/s3_loop_cfg3.log 2>&1; tail -2 gpurun_out/s3_loop_cfg3.log
