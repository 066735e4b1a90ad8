#!/bin/bash
# A/B of the DMMA kernel (kernel 4) against the ax8s/ax8c3 default (kernel 0)
# for every N=7 (equation, source, n_col): parity vs the oracle + timing.
for spec in "poisson trilinear 1" "poisson trilinear-partial 1" "poisson parallelepiped 1" "poisson stored 1" \
            "helmholtz trilinear 1" "helmholtz trilinear-merged 1" "helmholtz parallelepiped 1" "helmholtz stored 1" \
            "poisson trilinear 3" "poisson parallelepiped 3" "poisson stored 3" "helmholtz trilinear 3" \
            "helmholtz trilinear-merged 3" "poisson trilinear-partial 3"; do
  set -- $spec
  mesh=128,128,96; [ "$3" = 3 ] && mesh=128,128,32
  echo "== $1 $2 n_col=$3 mesh=$mesh"
  python tools/kernel_ab.py --equation $1 --source $2 --n-col $3 --mesh $mesh --cases 0:0,4:0 --rounds 3 2>&1 | grep -v "^$"
done
