# A/B: working tree vs _variants/$V, Poisson c1 sweep over orders $O (tools/ab_parse.py reads the log)
for r in 1 2; do
  echo "== new"; python tools/order_sweep.py --orders $O --variants ${VARS:-trilinear} --no-cpu --reps 10 2>&1 | grep "^N="
  echo "== $V"; HX_AXLOCAL_LIB=_variants/$V/libhx_axlocal.so python tools/order_sweep.py --orders $O --variants ${VARS:-trilinear} --no-cpu --reps 10 2>&1 | grep "^N="
done
