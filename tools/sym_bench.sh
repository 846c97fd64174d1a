#!/bin/bash
# symmetric mutual executors (fmm_p2p_sym, fmm_m2l_sym): tests, then C2 step
# timings directed vs symmetric per grain and precision (m2l / p2p stream spans)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_mutual.py -x -q > gpurun_out/sym_test.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/sym_test.log
for prec in ${PRECS:-fp32 fp64}; do
  for g in ${GRAINS:-5000 100000 1000000000}; do
    for sym in "" "--symmetric"; do
      echo "== $prec grain=$g $sym"
      python bench.py --mutual $sym --task-grain $g --precision $prec --steps 5 --warmup 5 --no-cpu-baseline --no-e2e 2> gpurun_out/sym_err.log | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(json.dumps({k: d.get(k) for k in ('value', 'ms_per_step', 'p2p_pairs', 'm2l_calls', 'stream_spans_ms', 'accuracy')}))
"
      tail -3 gpurun_out/sym_err.log
    done
  done
done
