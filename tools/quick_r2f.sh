O=gpurun_out
timeout 900 python -m pytest tests/test_data_parallel_gpu.py -q -x > $O/tests_r2f.txt 2>&1; tail -30 $O/tests_r2f.txt
