timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k grouped > gpurun_out/pytest_grouped.log 2>&1; echo pytest=$? 
P="python tools/spmm_probe.py --reps 3"
$P --config c2 > gpurun_out/t_c2_g4.json 2>gpurun_out/t.err
$P --config c2m --row-group 2 --ppl 2 > gpurun_out/t_c2m_g2_l1.json 2>>gpurun_out/t.err
tail -3 gpurun_out/t.err
