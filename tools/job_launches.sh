CMD="python bench.py --config ${CFG:-C2} ${EXTRA} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-accuracy"
$CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG:-C2}.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo rc=$?
