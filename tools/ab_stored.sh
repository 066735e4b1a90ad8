for r in 1 2 3; do
  echo "== new"; python tools/order_sweep.py --orders 5,6 --variants stored --no-cpu --reps 20 2>&1 | grep "^N="
  echo "== head"; HX_AXLOCAL_LIB=_variants/head/libhx_axlocal.so python tools/order_sweep.py --orders 5,6 --variants stored --no-cpu --reps 20 2>&1 | grep "^N="
done
