timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
bash tools/job_c4.sh
