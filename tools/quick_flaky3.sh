timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_reference_suite_gpu.py::test_reference_operator_and_trainer_cases_on_b200 > gpurun_out/tests_pre.txt 2>&1; tail -1 gpurun_out/tests_pre.txt
for i in 1 2 3; do timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -E "FAIL\]|test cases" | head -3; done
for i in 1 2 3; do D2FT_NO_SIDE=1 timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -E "FAIL\]|test cases" | head -3; done
for i in 1 2 3; do timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -E "FAIL\]|test cases" | head -3; done
