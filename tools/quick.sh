#!/bin/bash
# Quick GPU iteration: GPU tests (optionally a subset) + one bench line.
# usage (on the box): bash tools/quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-}
O=gpurun_out
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > $O/tests_$TAG.txt 2>&1
else timeout 900 python -m pytest tests -m gpu -q -x > $O/tests_$TAG.txt 2>&1; fi
tail -3 $O/tests_$TAG.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench_$TAG.json 2> $O/bench_$TAG.err || tail -20 $O/bench_$TAG.err
python - $O/bench_$TAG.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("value",round(d["value"],1),"ms",round(d["ms_per_step"],3),"e2e",round(d["e2e"]["value"],1))
    print("phase", d.get("phase_ms"))
    print("roofline", d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"]["active_head_gemms"])
except Exception as e: print("bench parse failed", e)
PY
