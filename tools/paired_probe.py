"""ncu target for the paired half-warp schedule: the adjoint and forward K6
at N^2 x N views (N=1024 default), 16 slices, built per XCT_FMTD_PAIRED mode.

  MODES="0 adjoint all" ncu --kernel-name regex:spmm --metrics \
    gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,\
    l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum python tools/paired_probe.py
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2009_07226_b200 import geometry, pipeline
n = int(os.environ.get("N", "1024"))
S = int(os.environ.get("S", "16"))
g = geometry.make_geometry(n, S, n)
rng = np.random.default_rng(0)
x = rng.random((g.num_voxels, S)).astype(np.float32)
y = rng.random((g.num_rays, S)).astype(np.float32)
for mode in os.environ.get("MODES", "0 adjoint all").split():
    os.environ["XCT_FMTD_PAIRED"] = mode
    s = pipeline.assemble(g, pipeline.SystemConfig(precision="mixed", ffactor=16))
    for _ in range(int(os.environ.get("REPS", "2"))):
        s.apply_adjoint(y)
        s.apply_forward(x)
    torch.cuda.synchronize()
    print("mode", mode, "done", flush=True)
    del s
    torch.cuda.empty_cache()
