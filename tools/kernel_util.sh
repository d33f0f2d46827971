#!/bin/bash
# Per-kernel tensor-pipe utilisation and SM-active fraction over one step.
# usage (on the box): bash tools/kernel_util.sh TAG
TAG=${1:-u}; O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/util_$TAG.csv python tools/profile_step.py 1 > /dev/null 2>&1
python tools/util_summary.py $O/util_$TAG.csv > $O/util_$TAG.txt; cat $O/util_$TAG.txt
