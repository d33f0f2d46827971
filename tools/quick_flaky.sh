O=gpurun_out
for i in 1 2 3; do
  timeout 300 python -m pytest tests/test_sched_gpu.py -q -x -k golden 2>&1 | tail -1
  timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | tail -1
done
timeout 600 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -B3 FAIL | head
