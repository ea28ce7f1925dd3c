#!/usr/bin/env python
"""Every kernel of libxct_b200 once, at a small size, for compute-sanitizer
(memcheck / racecheck / synccheck; one tool per run):

  compute-sanitizer --tool racecheck --kernel-name-exclude kns=at::,kns=void_at \\
      python tools/sanitize_small.py

K1/K2 Siddon, K11 matrix-free projector, K4 device transpose, K5 device
format build (ranges / count / fill, exact and fast schedules), K6 staged
SpMM in all four precisions (one row per lane set and grouped rows), K7-K9
normalization / CGLS updates / dots, the row-block measurement upload and
result download, and the K10 exchange kernels."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2009_07226_b200 import _lib, geometry, pipeline, solver  # noqa: E402


def main():
    dev = geometry.device()
    st = _lib.stream_handle(dev)
    g = geometry.make_geometry(48, 16, 32)
    A = geometry.build_system_matrix(g)                       # K1/K2
    vol = geometry.generate_phantom("random-blobs", 32, 16, seed=1)
    y = geometry.simulate_measurements(A, vol).slices_as_columns()
    x16 = torch.rand((g.num_voxels, 16), device=dev)
    geometry.project_matrix_free_f32(g, x16)                   # K11
    geometry.project_matrix_free_f32(g, torch.rand((g.num_rays, 16), device=dev), adjoint=True)
    for prec, order, rg in (("mixed", "native", None), ("single", "native", None),
                            ("single", "native", 1), ("double", "native", None),
                            ("half", "native", None), ("mixed", "reference", None),
                            ("single", "traversal", None)):
        cfg = pipeline.SystemConfig(precision=prec, ffactor=16, order=order, row_group=rg)
        sysm = pipeline.assemble(g, cfg)                       # K5 (device or host), K6
        res = solver.cgls_solve(sysm, y, solver.SolveConfig(max_iters=2, precision=prec))
        assert np.all(np.isfinite(res.x))
        sysm.apply_forward(vol.slices_as_columns().astype(np.float32))
        print(prec, order, rg, "ok", flush=True)
    # streamed device build (K4 band transpose, K5 fill) and host-tensor inputs
    pipeline.StreamedAssembly.CHUNK_NNZ = 2e4
    pipeline.StreamedAssembly.BAND_NNZ_DEV = 3e4
    s2 = pipeline.assemble(g, pipeline.SystemConfig(precision="mixed", ffactor=16,
                                                    build="streamed"))
    solver.cgls_solve(s2, torch.from_numpy(y.astype(np.float32)).pin_memory(),
                      solver.SolveConfig(max_iters=2, precision="mixed"))
    # K10
    C, n, fd = 2, 64, 16
    src = torch.rand((C, n, fd), device=dev)
    idx = torch.arange(0, n, 2, dtype=torch.int32, device=dev)
    out = torch.empty((C, idx.numel(), fd), device=dev)
    _lib.call("xct_gather_rows", src.data_ptr(), n, idx.data_ptr(), idx.numel(), C, fd, 0,
              out.data_ptr(), st)
    _lib.call("xct_accumulate_rows", src.data_ptr(), n, out.data_ptr(), idx.data_ptr(),
              idx.numel(), C, fd, 0, st)
    em = torch.empty((idx.numel(), C, fd), device=dev)
    _lib.call("xct_gather_records", src.data_ptr(), n, idx.data_ptr(), idx.numel(), 0, C, fd * 4,
              em.data_ptr(), st)
    _lib.call("xct_accumulate_records", src.data_ptr(), n, 0, em.data_ptr(), idx.data_ptr(),
              idx.numel(), C, fd, 0, st)
    fac = torch.ones(C, dtype=torch.float64, device=dev)
    scratch = torch.empty(148 * 8 + 8, dtype=torch.float64, device=dev)
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    _lib.call("xct_scale_chunks", src.data_ptr(), n * fd, C, fac.data_ptr(), 0,
              scratch.data_ptr(), ss.data_ptr(), st)
    torch.cuda.synchronize()
    print("all kernels ran", flush=True)


if __name__ == "__main__":
    main()
