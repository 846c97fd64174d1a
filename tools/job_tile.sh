timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/t.log
bash tools/job_ab.sh default w10s2 old > gpurun_out/ab.log 2>&1
for c in C1 C5; do python tools/p2p_bench.py --config $c 2>&1 | tail -1 >> gpurun_out/ab.log; FMM_B200_LIB=$PWD/paper_1209_3516_b200/libfmm_b200_old.so python tools/p2p_bench.py --config $c 2>&1 | tail -1 >> gpurun_out/ab.log; done
CMD2="python tools/p2p_bench.py --config C2 --reps 2"
$CMD2 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:p2p_f32 -s 3 -c 1 -o gpurun_out/bal_p2p_c2 $CMD2 > gpurun_out/ncu_c2.log 2>&1
echo rc=$? >> gpurun_out/ab.log
