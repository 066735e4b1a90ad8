# Helmholtz / n_col=3 / partial / merged at the role orders: roles vs -DHX_NO_ROLES
P="h:trilinear:0,c3:trilinear:0,h:c3:trilinear:0,trilinear-partial:0,h:trilinear-merged:0,h:parallelepiped:0,c3:parallelepiped:0,h:stored:0"
for o in "4 92,92,92" "5 77,77,77" "9 46,46,46" "13 33,33,33" "14 31,31,31" "15 29,29,29"; do
  set -- $o
  for r in 1 2; do
    echo "== roles N=$1"; python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
    echo "== noroles N=$1"; HX_AXLOCAL_LIB=_variants/noroles/libhx_axlocal.so python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
  done
done
