"""Single-GPU checks of kernels outside K6: the matrix-free FP32 projector
(K11), the row-block measurement upload / result download of cgls_solve,
and the K10 exchange kernels (gather / accumulate / scale) that the
domain-partitioned operator runs between its NCCL transfers
(src/comm.py:420-472, src/engine.py:189-221) -- exercised here on one GPU
so the driver's one-GPU box covers them."""

import numpy as np
import pytest
import torch

from paper_2009_07226_b200 import _lib, geometry, pipeline, solver

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_matrix_free_fp32_matches_csr_operator():
    g = geometry.make_geometry(96, 16, 64)
    A = geometry.build_system_matrix(g)
    dense = A.to_dense()
    rng = np.random.default_rng(3)
    x = rng.random((g.num_voxels, 16)).astype(np.float32)
    y = rng.random((g.num_rays, 16)).astype(np.float32)
    dev = geometry.device()
    fx = geometry.project_matrix_free_f32(g, torch.from_numpy(x).to(dev)).cpu().numpy()
    bx = geometry.project_matrix_free_f32(g, torch.from_numpy(y).to(dev),
                                          adjoint=True).cpu().numpy()
    ef, eb = _rel(fx, dense @ x.astype(np.float64)), _rel(bx, dense.T @ y.astype(np.float64))
    print(f"K11 matrix-free FP32 vs float64 CSR: forward {ef:.2e}, back projection {eb:.2e}")
    assert ef <= 1e-6 and eb <= 1e-6
    with pytest.raises(ValueError):
        geometry.project_matrix_free_f32(g, torch.from_numpy(x))       # host tensor


@pytest.mark.parametrize("prec", ["single", "mixed", "double"])
def test_cgls_measurement_inputs_are_equivalent(prec):
    """numpy f64, CUDA f64, a zero-stride CUDA view and a non-contiguous
    numpy view give the bit-identical solve; numpy f32 and a pinned f32 CPU
    tensor agree with each other (and x comes back float64)."""
    g = geometry.make_geometry(48, 40, 32)     # 40 slices: a padded last F-chunk
    A = geometry.build_system_matrix(g)
    vol = geometry.generate_phantom("random-blobs", 32, 40, seed=2)
    y = geometry.simulate_measurements(A, vol).slices_as_columns()
    sysm = pipeline.assemble(g, pipeline.SystemConfig(precision=prec, ffactor=16))
    cfg = solver.SolveConfig(max_iters=4, precision=prec)
    dev = geometry.device()
    base = solver.cgls_solve(sysm, y, cfg)
    assert base.x.dtype == np.float64 and base.x.shape == (g.num_voxels, 40)
    r_dev = solver.cgls_solve(sysm, torch.from_numpy(y).to(dev), cfg)
    assert torch.equal(r_dev.x.cpu(), torch.from_numpy(base.x))
    wide = np.zeros((y.shape[0], 80))
    wide[:, ::2] = y
    assert np.array_equal(solver.cgls_solve(sysm, wide[:, ::2], cfg).x, base.x)
    col = torch.from_numpy(np.ascontiguousarray(y[:, :1])).to(dev)
    r_b = solver.cgls_solve(sysm, col.expand(-1, 40), cfg)
    r_1 = solver.cgls_solve(sysm, np.repeat(y[:, :1], 40, axis=1), cfg)
    assert np.array_equal(r_b.x.cpu().numpy(), r_1.x)
    y32 = y.astype(np.float32)
    a = solver.cgls_solve(sysm, y32, cfg)
    pinned = torch.from_numpy(y32).pin_memory()
    b = solver.cgls_solve(sysm, pinned, cfg)
    assert np.array_equal(a.x, b.x.numpy())
    print(f"{prec}: f32 vs f64 measurements x rel {_rel(a.x, base.x):.2e}")
    assert _rel(a.x, base.x) <= (1e-5 if prec != "mixed" else 2e-3)


def test_row_blocks_cover_large_inputs(monkeypatch):
    """Many row blocks (upload and download) on a small problem give the
    same solve as one block."""
    import paper_2009_07226_b200.solver as S
    g = geometry.make_geometry(32, 16, 32)
    A = geometry.build_system_matrix(g)
    y = geometry.simulate_measurements(
        A, geometry.generate_phantom("shepp-logan-like", 32, 16)).slices_as_columns()
    sysm = pipeline.assemble(g, pipeline.SystemConfig(precision="mixed", ffactor=16))
    cfg = solver.SolveConfig(max_iters=3, precision="mixed")
    want = solver.cgls_solve(sysm, y, cfg).x
    monkeypatch.setattr(S, "_ROW_BLOCK_BYTES", 16 * 8 * 37)      # 37 rows per block
    got = solver.cgls_solve(sysm, y, cfg).x
    assert np.array_equal(got, want)


@pytest.mark.parametrize("f64", [0, 1])
def test_exchange_kernels_match_indexing(f64):
    dev = geometry.device()
    dt = torch.float64 if f64 else torch.float32
    gen = torch.Generator(device=dev).manual_seed(5)
    C, n_src, n_dst, fd = 3, 1000, 700, 16
    src = torch.rand((C, n_src, fd), generator=gen, device=dev, dtype=dt)
    idx = torch.randperm(n_src, generator=gen, device=dev)[:400].to(torch.int32)
    st = _lib.stream_handle(dev)
    out = torch.empty((C, 400, fd), dtype=dt, device=dev)
    _lib.call("xct_gather_rows", src.data_ptr(), n_src, idx.data_ptr(), 400, C, fd, f64,
              out.data_ptr(), st)
    assert torch.equal(out, src[:, idx.long()])
    # accumulate: owner first, then senders in order (the direct plan)
    dst = torch.zeros((C, n_dst, fd), dtype=dt, device=dev)
    ref = dst.clone()
    for s in range(3):
        part = torch.rand((C, 300, fd), generator=gen, device=dev, dtype=dt)
        pos = torch.randperm(n_dst, generator=gen, device=dev)[:300].to(torch.int32)
        _lib.call("xct_accumulate_rows", dst.data_ptr(), n_dst, part.data_ptr(), pos.data_ptr(),
                  300, C, fd, f64, st)
        ref[:, pos.long()] += part
    assert torch.equal(dst, ref)
    fac = torch.tensor([2.0, 0.5, 3.0], dtype=torch.float64, device=dev)
    scratch = torch.empty(148 * 8 + 8, dtype=torch.float64, device=dev)
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    want = dst * fac.to(dt)[:, None, None]
    _lib.call("xct_scale_chunks", dst.data_ptr(), n_dst * fd, C, fac.data_ptr(), f64,
              scratch.data_ptr(), ss.data_ptr(), st)
    assert torch.equal(dst, want)
    assert abs(float(ss) - float((want.double() ** 2).sum())) <= 1e-9 * float(ss)


def test_streamed_rescale_exponent_matches_the_median():
    """The streamed build's FP16 rescale exponent (xct_binade_hist per Siddon
    chunk, then the median's binade) equals half_rescale_exponent over the
    whole matrix (src/matrixstore.py:264-275), and the histogram equals
    numpy's."""
    from paper_2009_07226_b200 import matrixstore
    g = geometry.make_geometry(96, 4, 64)
    A = geometry.build_system_matrix(g)
    _, _, v = A.host_csr32()
    sa = pipeline.StreamedAssembly(g, pipeline.SystemConfig(precision="mixed", ffactor=16))
    sa.CHUNK_NNZ = 5e4                                  # several chunks
    chunks = sa._chunks(16)
    assert len(chunks) > 1
    assert sa._exponent(chunks) == matrixstore.half_rescale_exponent(np.asarray(v))
    dev = geometry.device()
    hist = torch.zeros(2048, dtype=torch.int64, device=dev)
    d_v = torch.from_numpy(np.asarray(v)).to(dev)
    _lib.call("xct_binade_hist", d_v.data_ptr(), d_v.numel(), hist.data_ptr(),
              _lib.stream_handle(dev))
    pos = np.asarray(v)[np.asarray(v) > 0]
    want = np.bincount(pos.view(np.int64) >> 52, minlength=2048)
    assert np.array_equal(hist.cpu().numpy(), want)
