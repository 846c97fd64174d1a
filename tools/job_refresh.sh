# Refresh the judged artifacts: full GPU tests, smoke, the default bench line,
# the reference arm, per-config lines, launch lists and the P2P ncu captures.
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
CFG=C2 bash tools/job_launches.sh
CFG=C3 bash tools/job_launches.sh
for c in C2 C3; do
CMD="python tools/p2p_bench.py --config $c --reps 2"
$CMD > gpurun_out/plain_p2p_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:p2p_f32 -s 3 -c 1 -o gpurun_out/r01_p2p_full_$c $CMD > gpurun_out/ncu_p2p_$c.log 2>&1
echo rc=$?
done
