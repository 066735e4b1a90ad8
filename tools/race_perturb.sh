#!/bin/bash
# Build the timing-perturbation library (every barrier jittered, -DHX_PERTURB,
# hx_common.cuh) as _variants/perturb/libhx_axlocal.so.  tools/sanitize_cases.py
# --dump then runs every kernel family with the normal and the perturbed
# library and compares the outputs bitwise (the race check of this pool, where
# compute-sanitizer is unavailable).
set -e
cd "$(dirname "$0")/.."
objs=$(ls build/obj/*.o | xargs -n1 basename | sed 's/\.o$//' | grep -v capi)
tools/build_variant.sh perturb "-DHX_PERTURB" $objs
rm -f _variants/perturb/*.o
