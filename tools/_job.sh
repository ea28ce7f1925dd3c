TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513"
timeout 1500 $TR bench.py --gpus 4 --config c3 --no-cpu-baseline > gpurun_out/bench_c3_n4.log 2>&1; echo c3=$?
grep metric gpurun_out/bench_c3_n4.log | cut -c1-300
timeout 2400 $TR bench.py --gpus 4 --config c5 --partition domain --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_dom4_v16.log 2>&1; echo c5=$?
grep metric gpurun_out/bench_c5_dom4_v16.log | cut -c1-300
