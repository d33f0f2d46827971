timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 ./oracle/_ref/test_b200_model_trainer > gpurun_out/memcheck_trainer.txt 2>&1; tail -25 gpurun_out/memcheck_trainer.txt
