timeout 600 python scripts/time_twoscale.py gpurun_out/s3_twoscale.json 2>&1 | tail -5
