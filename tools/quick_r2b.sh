O=gpurun_out
timeout 600 python -m pytest tests/test_dataset_gpu.py tests/test_step_gpu.py -q -x -k "units or nonfinite" > $O/tests_r2b.txt 2>&1; tail -15 $O/tests_r2b.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r2b.txt 2>&1; tail -3 $O/smoke_r2b.txt
timeout 600 python bench.py --no-cpu-baseline --no-vitl > $O/bench_r2b.json 2> $O/bench_r2b.err; python -c "
import json;d=json.load(open('$O/bench_r2b.json'));print(d['value'], json.dumps(d['e2e']))"; tail -3 $O/bench_r2b.err
