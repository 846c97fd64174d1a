# Bench lines only: default C2 (as the driver runs it), per-config and
# per-strategy lines, the reference arm.
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in C1 C3 C5; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --strategy treecode --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_treecode.json 2> gpurun_out/bench_tc.err
python bench.py --strategy listfmm --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_listfmm.json 2> gpurun_out/bench_lf.err
python bench.py --mutual --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_mutual.json 2> gpurun_out/bench_mu.err
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
