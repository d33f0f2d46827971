# ncu of the scheduler kernels (round 2): ViT-B step shape (profile_step.py) and
# the 144 x 1024 sweep at r = 0.25 / 1 (sched_one.py)
O=gpurun_out
M=gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max,smsp__inst_executed.sum,smsp__average_warp_latency_per_inst_issued.ratio
timeout 300 ncu --set full --clock-control none -k regex:"knapsack_kernel|compact_cols_kernel|plan_kernel" --launch-skip 3 --launch-count 3 -o $O/sched_vitb_r2 python tools/profile_step.py 1 > /dev/null 2>&1
ncu -i $O/sched_vitb_r2.ncu-rep --page raw --csv --metrics $M > $O/sched_vitb_r2.csv 2>&1
for r in 0.25 1; do
timeout 300 ncu --set full --clock-control none -k regex:knapsack_kernel --launch-skip 1 --launch-count 1 -o $O/sched_sweep_$r python tools/sched_one.py $r 2 > /dev/null 2>&1
ncu -i $O/sched_sweep_$r.ncu-rep --page raw --csv --metrics $M > $O/sched_sweep_$r.csv 2>&1
done
ls -la $O/*.csv | tail -4
