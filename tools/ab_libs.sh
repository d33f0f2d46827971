#!/bin/bash
# A/B of prebuilt variant libraries (build/var/NAME) and env settings on the
# bench value: usage bash tools/ab_libs.sh "name[:ENV=1 ...]" ...  ("" = in-tree)
for i in 1 2; do
for spec in "$@"; do
  n=${spec%%:*}; e=""; [[ "$spec" == *:* ]] && e=${spec#*:}
  lib=""; [ -n "$n" ] && [ -d build/var/$n ] && lib="D2FT_B200_LIB=build/var/$n/libd2ft_b200.so"
  env $lib $e timeout 300 python bench.py --no-cpu-baseline --no-vitl --steps 20 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec', round(d['ms_per_step'],4), round(d['e2e']['value'],1))"
done; done
