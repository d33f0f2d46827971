#!/bin/bash
# One measurement pass on the GPU box: tests, bench (both arms), launch list,
# and a full ncu capture of the dominant kernel (G1) for the roofline traffic.
# usage (from the repo root, on the box): bash tools/round_measure.sh TAG
TAG=${1:-run}
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/tests_$TAG.txt 2>&1; tail -3 $O/tests_$TAG.txt
timeout 600 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; cat $O/bench_$TAG.json
timeout 600 python bench.py --impl reference > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; cat $O/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
  python tools/profile_step.py 2 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_$TAG.csv 3 > $O/launches_$TAG.txt; head -30 $O/launches_$TAG.txt
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:G1<" \
  --launch-skip 3 --launch-count 1 -o $O/g1_full_$TAG python tools/profile_step.py 1 > /dev/null 2>&1
ncu -i $O/g1_full_$TAG.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  > $O/g1_traffic_$TAG.csv 2>/dev/null; cat $O/g1_traffic_$TAG.csv | tail -2
