#!/bin/bash
# Build named experiment variants of the library on the box (build/var/NAME).
# usage: bash tools/var_build.sh name1:"-DFOO=1" name2:"-DBAR" ...
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  make -s -j32 OBJDIR=build/var/$name/obj LIB=build/var/$name/libd2ft_b200.so EXTRA="$flags" \
    build/var/$name/libd2ft_b200.so > build_$name.log 2>&1 || { echo "build $name failed"; tail -5 build_$name.log; }
done
