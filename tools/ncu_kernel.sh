#!/bin/bash
# Full ncu capture (with source) of one launch of each named kernel in the step.
# usage (on the box): bash tools/ncu_kernel.sh TAG regex1 [regex2 ...]
TAG=$1; shift
O=gpurun_out
for k in "$@"; do
  n=$(echo "$k" | tr -cd 'A-Za-z0-9_')
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" \
    --launch-skip 3 --launch-count 1 -o $O/${n}_$TAG python tools/profile_step.py 1 > /dev/null 2>&1
  ncu -i $O/${n}_$TAG.ncu-rep --page source --csv --print-source sass > $O/${n}_$TAG.src.csv 2>/dev/null
  ncu -i $O/${n}_$TAG.ncu-rep --page raw --csv > $O/${n}_$TAG.raw.csv 2>/dev/null
  echo "$k done"
done
