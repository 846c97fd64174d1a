timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err; tail -2 gpurun_out/bench6.err
python -c "import json; d=json.load(open('gpurun_out/bench6.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_ms'], d['phase_ms'], d['e2e']['value'], d['gpu_launches_per_step'])"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo ncu rc=$?
