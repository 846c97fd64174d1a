CMD="python bench.py --config C4 --p 10 --theta 0.4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/m2l_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:m2l_lanes -s 1 -c 1 -o gpurun_out/m2l_lanes_p10 $CMD > gpurun_out/ncu_m2l.log 2>&1
echo rc=$?
