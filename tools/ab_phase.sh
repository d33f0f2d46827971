#!/bin/bash
# Build variants (name:"flags") on the box, then per-phase times of each
# (plus the in-tree build) with tools/phase_times.py; prints one line per lib.
# usage: bash tools/ab_phase.sh PHASES name1:"-DA" name2:"-DB" ...
PH=$1; shift
bash tools/var_build.sh "$@"
run() { env $1 timeout 200 python tools/phase_times.py 20 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); ph=d['phase_ms']
print('%-12s step %.4f  ' % ('$2', d['ms_per_step']) + '  '.join('%s %.4f' % (k, ph[k]) for k in '$PH'.split(',')))"; }
run "" in-tree
for spec in "$@"; do n=${spec%%:*}; run "D2FT_B200_LIB=build/var/$n/libd2ft_b200.so" $n; done
