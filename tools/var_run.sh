python tools/phase_times.py
for v in "$@"; do D2FT_B200_LIB=build/var/$v/libd2ft_b200.so timeout 120 python tools/phase_times.py; done
