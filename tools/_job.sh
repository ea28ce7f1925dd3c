timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi.log 2>&1; echo pytest=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514"
XCT_EXCHANGE_PROFILE=1 timeout 2400 $TR bench.py --gpus 4 --config c5 --partition domain --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/bench_c5_dom4_prof2.log 2>&1; echo c5p=$?
grep "exchange" gpurun_out/bench_c5_dom4_prof2.log | tail -2
timeout 2400 $TR bench.py --gpus 4 --config c5 --partition domain --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_dom4_v18.log 2>&1; echo c5=$?
grep metric gpurun_out/bench_c5_dom4_v18.log | cut -c1-300
