#!/bin/bash
# j-plane kernel (kernel 5) against the current default (kernel 0) at orders 2 and 3,
# every source / equation, n_col 1, C3 sizes (~100 M DOF).
for o in 2 3; do
  e=$([ $o = 2 ] && echo 155,155,155 || echo 116,116,116)
  for eq in poisson helmholtz; do
    for src in trilinear trilinear-partial trilinear-merged parallelepiped stored; do
      [ $eq = poisson ] && [ $src = trilinear-merged ] && continue
      [ $eq = helmholtz ] && [ $src = trilinear-partial ] && continue
      echo "== N=$o $eq $src"
      python tools/kernel_ab.py --order $o --equation $eq --source $src --mesh $e --cases 0:0,5:0 --rounds 3 --subset 128 2>&1 | grep -E "GDOF|parity|rror"
    done
  done
done
