O=gpurun_out
timeout 600 python -m pytest tests/test_lora_gpu.py tests/test_partition_gpu.py -q -x > $O/tests_r2d.txt 2>&1; tail -30 $O/tests_r2d.txt
