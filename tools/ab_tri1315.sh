P="trilinear:0,trilinear-partial:0,c3:trilinear:0,h:trilinear:0"
for o in "12 33,33,33" "14 29,29,29"; do
  set -- $o
  for r in 1 2; do
    echo "== new N=$1"; python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
    echo "== $V N=$1"; HX_AXLOCAL_LIB=_variants/$V/libhx_axlocal.so python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
  done
done
