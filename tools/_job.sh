XCT_VERBOSE=1 timeout 900 python bench.py > gpurun_out/bench_c2_v14.log 2>&1; echo b=$?
python tools/spmm_probe.py --reps 3 --config c2m > gpurun_out/v_c2m_g1.json 2>gpurun_out/v.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
