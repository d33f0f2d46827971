#!/bin/bash
# Same-box A/B of the in-tree library against prebuilt ones under abtmp/NAME
# (graph step ms and the eager attention-backward phase), interleaved rounds.
# usage (on the box): bash tools/ab_abtmp.sh ROUNDS NAME...
R=$1; shift
for r in $(seq 1 $R); do
  for v in in-tree "$@"; do
    lib=""; [ $v != in-tree ] && lib="D2FT_B200_LIB=abtmp/$v/libd2ft_b200.so"
    env $lib timeout 300 python tools/phase_times.py 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['phase_ms']['attn_bwd'], d['phase_ms']['attn_fwd'])"
  done
done
