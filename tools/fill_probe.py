#!/usr/bin/env python
"""Device format fill (K5) for one chunk of c5 views, per schedule mode:
CUDA-event time of build_format_device for the forward (A) part of views
[0, K1) of the 2048^2 x 2048-view geometry, and for the back-projection
part of one band of voxel rows.

  MODES="0 all" python tools/fill_probe.py
"""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2009_07226_b200 import geometry, matrixstore, pipeline  # noqa: E402

n, K = 2048, 2048
K1 = int(os.environ.get("K1", "128"))
g = geometry.make_geometry(K, 16, n)
dev = geometry.device()
cfg = pipeline.SystemConfig(precision="mixed", ffactor=16)
rw = pipeline._rows_per_warp(cfg, kind="forward")
ip, ix, v = geometry.siddon_csr(g, 0, K1, dev)
for mode in os.environ.get("MODES", "0 all").split():
    os.environ["XCT_FMTD_PAIRED"] = mode
    plan = matrixstore.assign_forward_regimes(
        matrixstore.forward_plan(K, n, rw, cfg.warps_per_cta, 0, K1), g.angles, n)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        part = matrixstore.build_format_device(ip, ix, v, K1 * n, g.num_voxels, plan, "mixed", 16,
                                               -10, cfg.smem_budget_effective, True, n, n, dev)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    info = part.info
    print(f"mode {mode}: forward part of {K1} views: {dt:.3f} s, n_padded {info['n_padded']}, "
          f"groups {info['n_groups']}, paired {info.get('paired_merged_steps')}/"
          f"{info.get('paired_half_steps')} fallbacks {info.get('paired_fallback_halves')} "
          f"cycles paired-gather/paired-job/quarter-job/quarter-gather {info.get('phase')}",
          flush=True)
