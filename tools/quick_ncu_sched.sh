O=gpurun_out
timeout 300 ncu --set full --import-source on -k regex:knapsack_kernel --launch-skip 1 --launch-count 1 -o $O/knap_r025 python tools/sched_one.py 0.25 2 > /dev/null 2>&1
ncu -i $O/knap_r025.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__average_warp_latency_per_inst_issued.ratio,smsp__inst_executed.sum,sm__cycles_elapsed.avg > $O/knap_raw.csv 2>&1; cat $O/knap_raw.csv | tail -3
ncu -i $O/knap_r025.ncu-rep --page source --csv --print-source sass > $O/knap_src.csv 2>/dev/null; wc -l $O/knap_src.csv
