P="c3:trilinear:0,h:c3:trilinear:0,c3:trilinear-partial:0,h:c3:trilinear-merged:0,c3:parallelepiped:0,c3:stored:0"
for r in 1 2; do
  for v in new m4 regm4; do
    echo "== $v N=7"; if [ $v = new ]; then L=""; else L=_variants/$v/libhx_axlocal.so; fi
    HX_AXLOCAL_LIB=$L python tools/sweep.py --order 7 --mesh 128,128,32 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
  done
done
