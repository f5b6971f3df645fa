#!/bin/bash
# A/B of experiment builds on the bench workload: [CFG=c2] [OPTS="a=1 b=0,c=1"] tools/ab_libs.sh lib1 lib2 ...
# (a lib is variants/<name> or "main" = the in-tree build); every lib runs every option set, twice.
cfg=${CFG:-c2}
opts=${OPTS:-slice_major=1}
for rep in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = main ]; then unset CC_LIB; else export CC_LIB=$lib/libcc.so; fi
    echo "== $lib"
    timeout -s KILL 300 python tools/ab_options.py --config $cfg --reps ${REPS:-20} $opts 2>&1 | grep -v "^\s*$" | tail -4
  done
done
