for i in 1 2 3 4 5 6 7 8; do
  timeout 300 ./oracle/_ref/test_b200_model_trainer 2>&1 | grep -E "FAIL|test cases" | head -3
done
