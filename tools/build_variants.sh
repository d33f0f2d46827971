#!/bin/bash
# Experiment builds of the library with -D switches (profiling only; each
# variant is the same sm_100a library with one epilogue part disabled).
# usage: tools/build_variants.sh name1:"-DFOO -DBAR" name2:"-DBAZ" ...
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  make -s -j8 OBJDIR=build/var/$name/obj LIB=build/var/$name/libd2ft_b200.so EXTRA="$flags" \
    build/var/$name/libd2ft_b200.so > /dev/null
  echo "built build/var/$name ($flags)"
done
