# A/B of the list-stream priority on C2 / C3 / C5 (alternating, 3 rounds)
for r in 1 2 3; do
  for pr in 0 1; do
    for cfg in C2 C3 C5; do
      FMM_B200_LIST_PRIORITY=$pr python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-accuracy 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg prio=$pr', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms'].items()})"
    done
  done
done
