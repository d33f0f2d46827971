#!/bin/bash
# A/B of the side-stream variants (bench value), two rounds.
for i in 1 2; do
for v in none side side7 side7n; do
  case $v in none) E="D2FT_NO_SIDE=1";; side) E="D2FT_NO_SIDE_G7=1";; side7) E="";; side7n) E="D2FT_SIDE_CTAS=64";; esac
  env $E timeout 300 python bench.py --no-cpu-baseline --no-vitl --steps 20 > gpurun_out/ab_$v$i.json 2>gpurun_out/ab_$v$i.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$v$i.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['e2e']['value'],1), d.get('lora',{}).get('ms_per_step'))" || tail -3 gpurun_out/ab_$v$i.err
done; done
