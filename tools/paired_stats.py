"""Paired-schedule statistics of one device-built A^T (and A) format:
merged half-steps and conflicting placements per region.

  N=512 python tools/paired_stats.py
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2009_07226_b200 import geometry, matrixstore, pipeline  # noqa: E402

n = int(os.environ.get("N", "512"))
g = geometry.make_geometry(n, 1, n)
A = geometry.build_system_matrix(g)
ip, ix, v = A.host_csr32()
cfg = pipeline.SystemConfig(precision="mixed", ffactor=16, row_group=1)
rw = pipeline._rows_per_warp(cfg)
dev = geometry.device()
exp = matrixstore.half_rescale_exponent(np.asarray(v))
t_ip, t_ix, t_v = pipeline._transpose(ip, ix, v, g.num_rays, g.num_voxels)
os.environ.setdefault("XCT_FMTD_PAIRED", "all")
sides = [("adjoint", t_ip, t_ix, t_v, g.num_voxels, g.num_rays,
          matrixstore.adjoint_plan(n, n, rw, cfg.warps_per_cta)),
         ("forward", ip, ix, v, g.num_rays, g.num_voxels,
          matrixstore.assign_forward_regimes(matrixstore.forward_plan(n, n, rw, cfg.warps_per_cta),
                                             g.angles, n))]
only = os.environ.get("SIDES", "adjoint forward").split()
for kind, a, b, c, nr, nc, plan in sides:
    if kind not in only:
        continue
    B, nk = pipeline.key_shape(g, kind)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    da, db, dc = (torch.from_numpy(t).to(dev) for t in (a, b, c))
    ev0.record()
    part = matrixstore.build_format_device(da, db, dc, nr, nc, plan, "mixed", 16, exp,
                                           cfg.smem_budget_effective, True, B, nk, dev)
    ev1.record()
    torch.cuda.synchronize()
    i = part.info
    extra = ""
    if "paired_half_steps" in i:
        hs, mg = i["paired_half_steps"], i["paired_merged_steps"]
        uc, mc = i["paired_conflicts"]["quarter_steps"], i["paired_conflicts"]["merged_steps"]
        u = hs - mg - mc
        extra = f" modelled LDS wavefronts per half-step {(2 * u + uc + mg + 2 * mc) / hs:.3f}"
    print(kind, os.environ.get("XCT_FMTD_PAIRED_EXTRA", "0"),
          f"build {ev0.elapsed_time(ev1):.0f} ms, n_padded {i['n_padded']}, nnz {i['nnz']}",
          {k: i[k] for k in i if k.startswith("paired")}, extra, flush=True)
