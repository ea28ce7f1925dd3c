P="python tools/spmm_probe.py --reps 3 --config c2"
$P --warps 8 > gpurun_out/w_c2_w8.json 2>gpurun_out/w.err
$P --warps 8 --smem 65536 > gpurun_out/w_c2_w8_s64.json 2>>gpurun_out/w.err
$P --warps 16 --smem 65536 > gpurun_out/w_c2_w16_s64.json 2>>gpurun_out/w.err
tail -3 gpurun_out/w.err
