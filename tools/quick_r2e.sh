O=gpurun_out
timeout 300 python tools/sched_latency.py 2>&1 | tail -8
timeout 900 python -m pytest tests/test_sched_gpu.py tests/test_reference_suite_gpu.py tests/test_metrics_gpu.py -q -x > $O/tests_r2e.txt 2>&1; tail -3 $O/tests_r2e.txt
