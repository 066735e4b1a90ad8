P="c3:trilinear:0,h:c3:trilinear:0,c3:trilinear-partial:0,h:c3:trilinear-merged:0,c3:parallelepiped:0,h:c3:parallelepiped:0,c3:stored:0,h:c3:stored:0"
for r in 1 2; do
  echo "== new N=7"; python tools/sweep.py --order 7 --mesh 128,128,32 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
  echo "== $V N=7"; HX_AXLOCAL_LIB=_variants/$V/libhx_axlocal.so python tools/sweep.py --order 7 --mesh 128,128,32 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
done
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ncol3 or helmholtz or role_table" 2>&1 | tail -1
