# ax_low (N=1, 2) A/B against _variants/head
P="h:trilinear:0,c3:trilinear:0,h:c3:trilinear:0,trilinear-partial:0,h:trilinear-merged:0,h:parallelepiped:0,c3:parallelepiped:0"
for r in 1 2; do
  echo "== new"; python tools/order_sweep.py --orders 1,2 --variants trilinear,parallelepiped --no-cpu --reps 10 2>&1 | grep "^N="
  echo "== head"; HX_AXLOCAL_LIB=_variants/head/libhx_axlocal.so python tools/order_sweep.py --orders 1,2 --variants trilinear,parallelepiped --no-cpu --reps 10 2>&1 | grep "^N="
done
for o in "1 200,200,200" "2 150,150,150"; do
  set -- $o
  for r in 1 2; do
    echo "== new N=$1"; python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
    echo "== head N=$1"; HX_AXLOCAL_LIB=_variants/head/libhx_axlocal.so python tools/sweep.py --order $1 --mesh $2 --reps 10 --rounds 2 --pairs "$P" 2>&1 | grep GDOF
  done
done
python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
