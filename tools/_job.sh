XCT_FWD_WARP_VIEWS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k grouped > gpurun_out/pytest_grouped.log 2>&1; echo pytest=$?
XCT_FWD_WARP_VIEWS=1 python tools/spmm_probe.py --reps 3 --config c2 > gpurun_out/v2_c2_wv.json 2>gpurun_out/v2.err
tail -3 gpurun_out/v2.err
