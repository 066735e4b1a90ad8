for r in 1 2; do
  for v in new lowo6 lowo8; do
    echo "== $v"; if [ $v = new ]; then L=""; else L=_variants/$v/libhx_axlocal.so; fi
    HX_AXLOCAL_LIB=$L python tools/order_sweep.py --orders 2 --variants parallelepiped --no-cpu --reps 10 2>&1 | grep "^N="
    HX_AXLOCAL_LIB=$L python tools/sweep.py --order 2 --mesh 150,150,150 --reps 10 --rounds 2 --pairs "h:parallelepiped:0,c3:parallelepiped:0" 2>&1 | grep GDOF
  done
done
