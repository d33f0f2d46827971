for v in in-tree build/exp/old/libd2ft_b200.so build/exp/noepi/libd2ft_b200.so in-tree build/exp/old/libd2ft_b200.so; do
  if [ "$v" = in-tree ]; then timeout 120 python tools/phase_times.py 20; else D2FT_B200_LIB=$v timeout 120 python tools/phase_times.py 20; fi
done
