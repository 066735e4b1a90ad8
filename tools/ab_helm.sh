P="h:trilinear:0,h:c3:trilinear:0,h:trilinear-merged:0,h:parallelepiped:0,h:stored:0"
for o in "3 93,93,93" "4 77,77,77" "6 58,58,58" "8 46,46,46" "11 36,36,36" "13 29,29,29"; do
  set -- $o
  for r in 1 2; do
    echo "== new N=$1"; python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
    echo "== $V N=$1"; HX_AXLOCAL_LIB=_variants/$V/libhx_axlocal.so python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
  done
done
