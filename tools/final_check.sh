# round-end style validation on one GPU: GPU tests, smoke, bench (both arms), C3 sweep
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/order_sweep.py --json gpurun_out/order_sweep.json > gpurun_out/order_sweep.txt 2>&1
