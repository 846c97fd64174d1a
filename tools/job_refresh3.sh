# Refresh after traversal changes: GPU tests, smoke, bench lines, launch lists.
timeout 900 python -m pytest tests/ -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
bash tools/job_bench_all.sh
CFG=C2 bash tools/job_launches.sh
CFG=C3 bash tools/job_launches.sh
