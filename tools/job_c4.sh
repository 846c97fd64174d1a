for pt in "3 0.6" "6 0.4" "8 0.5" "10 0.3" "10 0.6"; do set -- $pt
python bench.py --config C4 --p $1 --theta $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4.json 2> gpurun_out/c4.err; tail -1 gpurun_out/c4.err
python -c "import json; d=json.load(open('gpurun_out/c4.json')); print('p=$1 th=$2', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in d['kernel_ms'].items()}, 'm2l', d['m2l_calls'])"
done
