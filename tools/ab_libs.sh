#!/bin/bash
# Same-box A/B of alternative library builds: tools/ab_libs.sh "<kernel_ab args>" lib1 lib2 ...
# (a lib path of "-" means the in-tree build); rounds interleaved across libraries.
args=$1; shift
for r in 1 2 3; do
  for lib in "$@"; do
    if [ "$lib" = "-" ]; then unset HX_AXLOCAL_LIB; else export HX_AXLOCAL_LIB=$lib; fi
    echo "== round $r lib $lib"
    python tools/kernel_ab.py $args --subset 64 2>&1 | grep "GDOF"
  done
done
