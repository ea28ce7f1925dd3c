TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512"
timeout 2400 $TR bench.py --gpus 4 --config c5 --partition domain --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_c5_dom4_w.log 2>&1; echo dom4=$?
grep metric gpurun_out/bench_c5_dom4_w.log | cut -c1-400
