O=gpurun_out
timeout 600 python -m pytest tests/test_step_gpu.py tests/test_reference_suite_gpu.py tests/test_prepass_gpu.py -q -x > $O/tests_r2c.txt 2>&1; tail -15 $O/tests_r2c.txt
