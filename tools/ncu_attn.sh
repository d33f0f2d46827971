#!/bin/bash
# ncu source-level capture of one attention-forward launch for the in-tree
# library and each named variant (build/var/NAME); summaries in gpurun_out/.
# usage: bash tools/ncu_attn.sh KERNEL_REGEX TAG [variant ...]
K=$1; TAG=$2; shift 2
O=gpurun_out
for v in in-tree "$@"; do
  lib=""; [ "$v" != in-tree ] && lib="D2FT_B200_LIB=build/var/$v/libd2ft_b200.so"
  env $lib timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" \
    --launch-skip 14 --launch-count 1 -o $O/${TAG}_$v python tools/profile_step.py 1 > /dev/null 2>&1
  ncu -i $O/${TAG}_$v.ncu-rep --page source --csv --print-source sass > $O/${TAG}_$v.src.csv 2>/dev/null
  ncu -i $O/${TAG}_$v.ncu-rep --page raw --csv > $O/${TAG}_$v.raw.csv 2>/dev/null
  python tools/ncu_src.py $O/${TAG}_$v.src.csv 25 > $O/${TAG}_$v.top.txt 2>&1
  echo "== $v"; head -30 $O/${TAG}_$v.top.txt
done
