timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err; tail -2 gpurun_out/bench6.err
python -c "import json; d=json.load(open('gpurun_out/bench6.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_ms'], d['phase_ms'], d['e2e']['value'], d['gpu_launches_per_step'])"
