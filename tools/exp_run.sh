#!/bin/bash
# Build experiment variants on the box and compare per-phase times.
# usage: bash tools/exp_run.sh name1:"-DFOO" name2:"-DBAR" ...
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  make -s -j16 OBJDIR=build/var/$name/obj LIB=build/var/$name/libd2ft_b200.so EXTRA="$flags" \
    build/var/$name/libd2ft_b200.so > /dev/null 2>&1 || echo "build $name failed"
done
timeout 120 python tools/phase_times.py 20
for spec in "$@"; do name=${spec%%:*}; D2FT_B200_LIB=build/var/$name/libd2ft_b200.so timeout 120 python tools/phase_times.py 20; done
