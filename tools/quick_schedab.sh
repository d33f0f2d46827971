for v in ldcg:"-DD2FT_SCHED_LDCG" nofence:"-DD2FT_SCHED_NOFENCE" both:"-DD2FT_SCHED_LDCG -DD2FT_SCHED_NOFENCE"; do
  name=${v%%:*}; flags=${v#*:}
  make -s -j16 OBJDIR=build/var/$name/obj LIB=build/var/$name/libd2ft_b200.so EXTRA="$flags" build/var/$name/libd2ft_b200.so > /dev/null 2>&1 || echo "build $name failed"
done
echo base; timeout 200 python tools/sched_latency.py 2>&1 | tail -4
for name in ldcg nofence both; do echo $name; D2FT_B200_LIB=build/var/$name/libd2ft_b200.so timeout 200 python tools/sched_latency.py 2>&1 | tail -4; done
