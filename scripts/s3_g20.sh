timeout 1500 python tests/report_configs.py gpurun_out/s3_configs_report.json > gpurun_out/s3_configs_report.log 2>&1; tail -5 gpurun_out/s3_configs_report.log
