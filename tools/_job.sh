python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench_c2_v19.log 2>&1; echo bench=$?
grep metric gpurun_out/bench_c2_v19.log | cut -c1-250
