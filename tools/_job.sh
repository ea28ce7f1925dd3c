TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515"
for W in 8 2; do
XCT_EXCHANGE_WAVES=$W timeout 2400 $TR bench.py --gpus 4 --config c5 --partition domain --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_dom4_w$W.log 2>&1; echo c5w$W=$?
grep metric gpurun_out/bench_c5_dom4_w$W.log | cut -c150-260
done
