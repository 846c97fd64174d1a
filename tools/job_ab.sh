# A/B the P2P kernel: variants given as args (default = the in-tree library)
for v in "$@"; do
  if [ $v = default ]; then L=""; else L=$PWD/paper_1209_3516_b200/libfmm_b200_$v.so; fi
  for c in C2 C3; do FMM_B200_LIB=$L python tools/p2p_bench.py --config $c 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', d['config'], round(d['ms'],3), round(d['tflops_20'],2), max(d['rel_l2_vs_fp64']))"; done
done
