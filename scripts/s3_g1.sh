set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3_tests.log 2>&1; tail -3 gpurun_out/s3_tests.log
timeout 300 python scripts/sweep_cfg4.py gpurun_out/s3_sweep.json --no-solve > gpurun_out/s3_sweep.log 2>&1; tail -12 gpurun_out/s3_sweep.log
timeout 120 python scripts/time_kernel.py cfg3 300
