for i in 1 2 3 4 5; do timeout 300 python -m pytest tests/test_data_parallel_gpu.py -q 2>&1 | grep -E "passed|failed|AssertionError|^E " | head -4; done
