O=gpurun_out
timeout 600 python -m pytest tests/test_step_gpu.py tests/test_parity_bench_gpu.py -q -x -k "dh64 or short or vitb" > $O/tests_af.txt 2>&1; tail -3 $O/tests_af.txt
make -s -j16 OBJDIR=build/var/cg1/obj LIB=build/var/cg1/libd2ft_b200.so EXTRA="-DD2FT_AF_CG=1" build/var/cg1/libd2ft_b200.so > /dev/null 2>&1 || echo "build failed"
for i in 1 2 3; do
  timeout 200 python tools/phase_times.py 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cg2', d['ms_per_step'], d['phase_ms']['attn_fwd'], d['phase_ms']['attn_bwd'])"
  D2FT_B200_LIB=build/var/cg1/libd2ft_b200.so timeout 200 python tools/phase_times.py 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cg1', d['ms_per_step'], d['phase_ms']['attn_fwd'], d['phase_ms']['attn_bwd'])"
done
