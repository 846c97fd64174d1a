CMD="python tools/p2p_bench.py --reps 3"
$CMD > gpurun_out/plain_p2p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:p2p_f32 -s 2 -c 1 -o gpurun_out/p2p_packed_prof $CMD > gpurun_out/ncu_p2p.log 2>&1
echo rc=$?
