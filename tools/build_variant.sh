#!/bin/bash
# Build an alternate libhx_axlocal.so with extra flags on some order-generic kernel
# objects, for A/B timing (load it with HX_AXLOCAL_LIB=<path>):
#   tools/build_variant.sh <tag> "<nvcc flags>" <n1> [<n1> ...]
# -> _variants/<tag>/libhx_axlocal.so (git-ignored, travels with gpurun) (default objects from `make` for everything else)
set -e
cd "$(dirname "$0")/.."
tag=$1; flags=$2; shift 2
make -s -j16 >/dev/null
d=_variants/$tag
mkdir -p "$d"
objs=()
for o in build/obj/*.o; do
  b=$(basename "$o" .o)
  hit=""
  for n in "$@"; do [ "$b" = "ax_fastn_$n" ] && hit=$n; done
  if [ -n "$hit" ]; then
    nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a \
      -Iinclude -DHX_N1="$hit" $flags -c paper_2504_07042_b200/csrc/ax_fastn.cu -o "$d/$b.o" &
    objs+=("$d/$b.o")
  else
    objs+=("$o")
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$d/libhx_axlocal.so" "${objs[@]}" -cudart static
echo "$d/libhx_axlocal.so"
