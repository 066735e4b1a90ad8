#!/bin/bash
# Build an alternate libhx_axlocal.so with extra nvcc flags on some objects, for A/B
# timing (load it with HX_AXLOCAL_LIB=<path>):
#   tools/build_variant.sh <tag> "<nvcc flags>" <object> [<object> ...]
# objects are build/obj basenames: ax_fast, setup, ax_fastn_<n1>, ax_generic_<n1>, ax_low_<n1>, ...
# -> _variants/<tag>/libhx_axlocal.so (git-ignored, travels with gpurun)
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
  for n in "$@"; do [ "$b" = "$n" ] && hit=1; done
  if [ -n "$hit" ]; then
    src=${b%_*}; n1=${b##*_}; extra=""; case $b in ax_mma|ax_plane_*) extra=-fmad=false;; esac
    case "$b" in
      ax_fastn_*|ax_generic_*|ax_low_*|ax_plane_*) def="-DHX_N1=$n1"; srcf=paper_2504_07042_b200/csrc/$src.cu ;;
      *) def=""; srcf=paper_2504_07042_b200/csrc/$b.cu ;;
    esac
    nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a \
      -Iinclude $def $flags $extra -c "$srcf" -o "$d/$b.o" &
    objs+=("$d/$b.o")
  else
    objs+=("$o")
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$d/libhx_axlocal.so" "${objs[@]}" -cudart static
echo "$d/libhx_axlocal.so"
