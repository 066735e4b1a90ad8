set -e
O=${O:-3,4,5,8,9,11,12,13,14,15}
for r in 1 2; do
  echo "== roles"; python tools/order_sweep.py --orders $O --no-cpu --reps 10 2>&1 | grep -v "^#"
  echo "== noroles"; HX_AXLOCAL_LIB=_variants/noroles/libhx_axlocal.so python tools/order_sweep.py --orders $O --no-cpu --reps 10 2>&1 | grep -v "^#"
done
python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
