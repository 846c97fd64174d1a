CMD="python bench.py --config C4 --p 10 --theta 0.6 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_m2l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:m2l_block -s 1 -c 1 -o gpurun_out/m2l_prof $CMD > gpurun_out/ncu_m2l.log 2>&1
echo rc=$?
