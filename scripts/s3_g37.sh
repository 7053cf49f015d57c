timeout 600 python scripts/time_loop_cfg3.py gpurun_out/s3_loop_cfg3_warm.json --warm > gpurun_out/s3_loop_warm.log 2>&1; tail -1 gpurun_out/s3_loop_warm.log
