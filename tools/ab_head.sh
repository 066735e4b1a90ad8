# A/B of the working tree against a library built from an older commit (_variants/head)
O=${O:-2,3,4,5,6,8,9,10,11,12,13,14,15}
for r in 1 2; do
  echo "== new"; python tools/order_sweep.py --orders $O --no-cpu --reps 10 2>&1 | grep "^N="
  echo "== ${V:-head}"; HX_AXLOCAL_LIB=_variants/${V:-head}/libhx_axlocal.so python tools/order_sweep.py --orders $O --no-cpu --reps 10 2>&1 | grep "^N="
done
P="h:trilinear:0,c3:trilinear:0,h:c3:trilinear:0,trilinear-partial:0,h:trilinear-merged:0,h:parallelepiped:0,c3:parallelepiped:0,h:stored:0,stored:0"
for o in ${HO:-"4 92,92,92" "5 77,77,77" "6 66,66,66" "9 46,46,46" "11 39,39,39" "15 29,29,29"}; do
  set -- $o
  for r in 1 2; do
    echo "== new N=$1"; python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
    echo "== ${V:-head} N=$1"; HX_AXLOCAL_LIB=_variants/${V:-head}/libhx_axlocal.so python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
  done
done
