for i in $(seq 1 15); do timeout 300 python -m pytest tests/test_data_parallel_gpu.py -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|^E  " | head -4; done
