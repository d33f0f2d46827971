O=gpurun_out
timeout 900 python -m pytest tests/test_step_gpu.py tests/test_parity_bench_gpu.py tests/test_prepass_gpu.py tests/test_lora_gpu.py -q -x -k "dh64 or short or vitb or vitl or lora" > $O/tests_ab.txt 2>&1; tail -3 $O/tests_ab.txt
for i in 1 2 3; do timeout 200 python tools/phase_times.py 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('new', d['ms_per_step'], d['phase_ms']['attn_fwd'], d['phase_ms']['attn_bwd'])"; done
