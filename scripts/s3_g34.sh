timeout 600 python -m pytest tests/test_gpu_configs.py -q -x -k "sampled_tight" 2>&1 | tail -15
