P="h:trilinear:0,c3:trilinear:0,h:c3:trilinear:0,trilinear-partial:0,h:trilinear-merged:0,h:parallelepiped:0,c3:parallelepiped:0,trilinear:0,parallelepiped:0"
for r in 1 2; do
  for v in new epb5all prev; do
    echo "== $v N=6"; if [ $v = new ]; then L=""; else L=_variants/$v/libhx_axlocal.so; fi
    HX_AXLOCAL_LIB=$L python tools/sweep.py --order 6 --mesh 66,66,66 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
  done
done
