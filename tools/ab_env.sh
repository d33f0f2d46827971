for i in 1 2; do
for v in none pdl side; do
  case $v in none) E="";; pdl) E="D2FT_PDL=1";; side) E="D2FT_NO_SIDE=1";; esac
  env $E timeout 300 python bench.py --no-cpu-baseline --no-vitl --steps 20 > gpurun_out/ab_$v$i.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$v$i.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['e2e']['value'])"
done; done
