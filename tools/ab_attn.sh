for i in 1 2 3; do
  timeout 200 python tools/phase_times.py 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('new', d['phase_ms']['attn_fwd'], d['phase_ms']['attn_bwd'])"
  D2FT_B200_LIB=build/var/old/libd2ft_b200.so timeout 200 python tools/phase_times.py 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('old', d['phase_ms']['attn_fwd'], d['phase_ms']['attn_bwd'])"
done
