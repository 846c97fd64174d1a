# ncu --set full of the list-construction kernels on C2 (plan_rows, row sort,
# scatter): one capture each, after the same command ran clean without ncu
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-accuracy"
$CMD > gpurun_out/plain_plan.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"plan_rows_kernel|row_sort_bitmap_kernel|row_scatter_kernel" -s 8 -c 4 -o gpurun_out/plan_prof $CMD > gpurun_out/ncu_plan.log 2>&1
echo rc=$?
