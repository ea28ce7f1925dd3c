timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python tools/spmm_probe.py --reps 3 --config c2 > gpurun_out/y_c2_ffma2.json 2>gpurun_out/y.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_v17.log 2>&1; echo bench=$?
grep metric gpurun_out/bench_c2_v17.log | cut -c1-250
