# Refresh the judged artifacts after a list/plan change (the P2P kernel's
# own ncu captures are unchanged): GPU tests, smoke, the default bench line,
# the reference arm, per-config and per-strategy lines, launch lists.
set -x
timeout 900 python -m pytest tests/ -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in C1 C3 C5; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --strategy treecode --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_treecode.json 2> gpurun_out/bench_tc.err
python bench.py --strategy listfmm --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_listfmm.json 2> gpurun_out/bench_lf.err
python bench.py --mutual --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_mutual.json 2> gpurun_out/bench_mu.err
CFG=C2 bash tools/job_launches.sh
CFG=C3 bash tools/job_launches.sh
