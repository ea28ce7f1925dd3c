timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi.log 2>&1; echo pytest=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516"
timeout 900 $TR bench.py --gpus 2 > gpurun_out/bench_c2_n2_v19.log 2>&1; echo n2=$?
timeout 900 $TR bench.py --gpus 2 --partition domain --no-cpu-baseline > gpurun_out/bench_c2_dom2_v19.log 2>&1; echo dom2=$?
grep metric gpurun_out/bench_c2_n2_v19.log | cut -c150-280; grep metric gpurun_out/bench_c2_dom2_v19.log | cut -c150-280
