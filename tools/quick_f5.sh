D2FT_NO_SIDE_G7=1 timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -E "epoch|FAIL\]|test cases"
D2FT_NO_SIDE_G7=1 D2FT_NO_GRAPH=1 timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -E "epoch|FAIL\]|test cases"
