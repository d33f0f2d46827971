timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 ./oracle/_ref/test_b200_model_trainer 2>&1 | tail -4
run() { n=0; f=0; for i in $(seq 1 $2); do n=$((n+1)); env $1 timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -q "failed: 0 " || f=$((f+1)); done; echo "$1 runs $n fails $f"; }
run "D2FT_NO_SIDE=1" 12
run "D2FT_NO_SIDE_G7=1" 8
run "X=1" 12
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_data_parallel_gpu.py tests/test_dataset_gpu.py -q -p no:cacheprovider 2>&1 | tail -1; done
