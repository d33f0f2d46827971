run() { n=0; f=0; for i in $(seq 1 $2); do n=$((n+1)); env $1 timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -q "failed: 0 " || f=$((f+1)); done; echo "$1 runs $n fails $f"; }
run "D2FT_NO_SIDE_G7=1" 4
run "X=1" 4
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tests_full_r2e.txt 2>&1; tail -3 gpurun_out/tests_full_r2e.txt
