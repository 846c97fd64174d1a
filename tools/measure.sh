#!/bin/bash
# One measurement pass on a gpurun box (outputs under gpurun_out/, copy the
# ones to keep into profiles/rNN_*):
#   bash tools/measure.sh bench     bench lines: C2 (driver default), C2 fp64, C1/C3/C5, strategies, reference arm
#   bash tools/measure.sh launches  ncu launch list of one C2 and one C3 bench step (gpu__time_duration per launch)
#   bash tools/measure.sh p2p       ncu --set full of the C2 P2P kernel (tools/p2p_bench.py)
#   bash tools/measure.sh p2p64     ncu --set full of the C2 FP64 P2P kernel (tools/p2p64_check.py)
#   bash tools/measure.sh m2l       grouped M2L timings (C4, p 7-10) and ncu --set full of m2l_dmma<10>
#   bash tools/measure.sh c4        the C4 accuracy/speed sweep, fp32 and fp64 (tools/c4_sweep.py)
# Each ncu pass runs only after the same command exited 0 without ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
case "$1" in
bench)
  python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
  python bench.py --precision fp64 --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_fp64.json 2> gpurun_out/bench_c2_fp64.err
  python bench.py --precision fp32acc --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_fp32acc.json 2> gpurun_out/bench_c2_fp32acc.err
  for c in C1 C3 C5; do
    python bench.py --config $c --steps 5 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  done
  for s in treecode listfmm; do
    python bench.py --strategy $s --steps 10 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2_$s.json 2> gpurun_out/bench_$s.err
  done
  python bench.py --mutual --steps 10 --no-cpu-baseline > gpurun_out/bench_c2_mutual.json 2> gpurun_out/bench_mu.err
  python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  ;;
launches)
  for c in C2 C3; do
    CMD="python bench.py --config $c --steps 1 --warmup 5 --no-cpu-baseline --no-e2e --no-accuracy"
    $CMD > gpurun_out/plain_$c.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$c.csv $CMD > gpurun_out/ncu_launches_$c.log 2>&1; echo "launches $c rc=$?"
  done
  ;;
p2p)
  CMD="python tools/p2p_bench.py --reps 3"
  $CMD > gpurun_out/plain_p2p.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:p2p_f32 \
    -s 2 -c 1 -o gpurun_out/p2p_prof -f $CMD > gpurun_out/ncu_p2p.log 2>&1; echo "p2p rc=$?"
  ;;
p2p64)
  CMD="python tools/p2p64_check.py --reps 2"
  $CMD > gpurun_out/plain_p2p64.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:p2p_f64s \
    -s 1 -c 1 -o gpurun_out/p2p64_prof -f $CMD > gpurun_out/ncu_p2p64.log 2>&1; echo "p2p64 rc=$?"
  ;;
m2l)
  # grouped M2L (DMMA) at the C4 corner: per-order timings, then ncu of the p=10 kernel
  for a in "--p 10 --theta 0.3" "--p 10 --theta 0.5" "--p 9 --theta 0.4" "--p 8 --theta 0.3" "--p 8 --theta 0.4" "--p 7 --theta 0.4"; do
    python tools/m2l_bench.py --config C4 $a --reps 5
  done > gpurun_out/m2l_grouped.log 2>&1
  CMD="python tools/m2l_bench.py --config C4 --p 10 --theta 0.3 --reps 1 --mode grouped"
  $CMD > gpurun_out/plain_m2l.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:m2l_dmma \
    -s 1 -c 1 -o gpurun_out/m2l_prof -f $CMD > gpurun_out/ncu_m2l.log 2>&1; echo "m2l rc=$?"
  ;;
c4)
  python tools/c4_sweep.py fp32 > gpurun_out/c4_fp32.log 2>&1
  python tools/c4_sweep.py fp64 > gpurun_out/c4_fp64.log 2>&1
  ;;
*) echo "usage: $0 bench|launches|p2p|p2p64|m2l|c4"; exit 2;;
esac
