# End-of-session refresh: GPU tests, smoke, bench lines (default C2 first,
# then the reference arm, per-config and per-strategy lines), launch lists,
# and the C4 accuracy/speed sweep in both precisions.
set -x
timeout 900 python -m pytest tests/ -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err
for c in C1 C3 C5; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --strategy treecode --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_treecode.json 2> gpurun_out/bench_tc.err
python bench.py --strategy listfmm --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_listfmm.json 2> gpurun_out/bench_lf.err
python bench.py --mutual --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_mutual.json 2> gpurun_out/bench_mu.err
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CFG=C2 bash tools/job_launches.sh
CFG=C3 bash tools/job_launches.sh
python tools/c4_sweep.py fp32 > gpurun_out/c4_fp32.log 2>&1
python tools/c4_sweep.py fp64 > gpurun_out/c4_fp64.log 2>&1
