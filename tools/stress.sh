#!/bin/bash
# Stress runs that found this round's races (run on the GPU box):
#   the operator/trainer binding suite under the stream-placement variants,
#   memcheck of it, and the data-parallel / Dataset GPU tests repeatedly.
#   usage: bash tools/stress.sh [repeats]
N=${1:-8}
run() { f=0; for i in $(seq 1 $2); do env $1 timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -q "failed: 0 " || f=$((f+1)); done; echo "$1: $2 runs, $f failed"; }
run "D2FT_DEFAULT=1" $N
run "D2FT_NO_SIDE=1" $N
run "D2FT_NO_SIDE_G7=1" $N
# memcheck only on request (some GPU pools close compute-sanitizer)
[ -n "$D2FT_STRESS_MEMCHECK" ] && timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 ./oracle/_ref/test_b200_model_trainer 2>&1 | tail -2
for i in $(seq 1 $N); do timeout 300 python -m pytest tests/test_data_parallel_gpu.py tests/test_dataset_gpu.py -q 2>&1 | tail -1; done
timeout 300 python tools/mode_probe.py 16 2>&1 | tail -9
