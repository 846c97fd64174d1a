CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_pf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:p2p_f32 -s 3 -c 1 -o gpurun_out/r01_p2p_full $CMD > gpurun_out/ncu_pf.log 2>&1
echo rc=$?
CMD2="python tools/p2p_bench.py --config C3 --reps 2"
$CMD2 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none -k regex:p2p_f32 -s 1 -c 1 -o gpurun_out/r01_p2p_full_c3 $CMD2 > gpurun_out/ncu_c3.log 2>&1
echo rc=$?
