timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
for c in C2 C3; do
python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -1 gpurun_out/bench_$c.err
python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['value'], d['ms_per_step'], round(d['roofline']['frac'],3), {k: round(v,2) for k,v in d['kernel_ms'].items()}, {k: round(v,2) for k,v in d['phase_ms'].items()})"
done
