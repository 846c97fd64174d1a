timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -2 gpurun_out/bench5.err
python -c "import json; d=json.load(open('gpurun_out/bench5.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_ms'], d['e2e'], d['clocks'], d['gpu_launches_per_step'])"
