for v in default s4; do
  if [ $v = default ]; then L=""; else L=$PWD/paper_1209_3516_b200/libfmm_b200_$v.so; fi
  FMM_B200_LIB=$L python tools/p2p_bench.py 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v C2', round(d['ms'],3), round(d['tflops_20'],2), d['rel_l2_vs_fp64'])"
  FMM_B200_LIB=$L python tools/p2p_bench.py --config C3 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v C3', round(d['ms'],3), round(d['tflops_20'],2), d['rel_l2_vs_fp64'])"
done
