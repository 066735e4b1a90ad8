P="h:trilinear-merged:0,h:trilinear:0,h:c3:trilinear:0"
for o in "11 36,36,36" "13 29,29,29" "14 27,27,27"; do
  set -- $o
  for r in 1 2; do
    echo "== new N=$1"; python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
    echo "== $V N=$1"; HX_AXLOCAL_LIB=_variants/$V/libhx_axlocal.so python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
  done
done
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "helmholtz or role_table or every_order" 2>&1 | tail -1
