"""The device format builder (K4/K5 on the GPU, csrc/format_device.cu)
against the host builder (format_build.cpp), byte for byte: same load
groups, same group maps, same bank schedule, same slab words -- and the
streamed device build of a whole operator against the monolithic host
build (replaces src/matrixstore.py:189-201, :250-262, :417-562)."""

import numpy as np
import pytest
import torch

from paper_2009_07226_b200 import _lib, geometry, matrixstore, pipeline

pytestmark = pytest.mark.gpu


def _host_words(hf, precision):
    """The host format's slab entries encoded as upload_format stores them."""
    slots = hf.arrays["slots"].astype(np.int64) & 0xFFFF
    off = slots << 4
    if precision in ("half", "mixed"):
        bits = hf.arrays["values"].view(np.uint16).astype(np.int64)
        return ((off << 16) | bits).astype(np.uint32).view(np.int32), None
    return hf.arrays["values"], off.astype(np.uint16).view(np.int16)


def _compare(hf, part, precision):
    for k in ("n_cta", "n_groups", "n_slots", "n_padded", "nnz", "max_group_slots",
              "underflow_count"):
        assert int(hf.info[k]) == int(part.info[k]), k
    assert float(hf.info["max_rel_quant_error"]) == pytest.approx(
        float(part.info["max_rel_quant_error"]), rel=0, abs=0)
    T = {k: v.cpu().numpy() for k, v in part.tensors.items()}
    for k in ("cta_group_ptr", "group_map_ptr", "group_map", "slab_off", "slab_width"):
        n = len(hf.arrays[k])
        assert np.array_equal(T[k][:n], hf.arrays[k]), k
    vals, slots = _host_words(hf, precision)
    n = int(hf.info["n_padded"])
    assert np.array_equal(T["values"][:n], vals), "slab values"
    assert not T["values"][n:].any()
    if slots is not None:
        assert np.array_equal(T["slots"][:n], slots), "slab slots"


CASES = [(96, 64, "mixed", True), (96, 64, "mixed", False), (180, 128, "mixed", True),
         (64, 48, "single", True), (64, 48, "double", True), (48, 40, "half", True)]


@pytest.mark.parametrize("k,n,precision,schedule", CASES)
def test_device_builder_equals_host_builder(k, n, precision, schedule):
    g = geometry.make_geometry(k, 1, n)
    A = geometry.build_system_matrix(g)
    ip, ix, v = A.host_csr32()
    cfg = pipeline.SystemConfig(precision=precision, ffactor=16, row_group=1)
    rw = pipeline._rows_per_warp(cfg)
    dev = geometry.device()
    exp = matrixstore.half_rescale_exponent(np.asarray(v)) if precision in ("half", "mixed") \
        else 0
    budget = cfg.smem_budget_effective
    t_ip, t_ix, t_v = pipeline._transpose(ip, ix, v, g.num_rays, g.num_voxels)
    sides = [("forward", ip, ix, v, g.num_rays, g.num_voxels,
              matrixstore.assign_forward_regimes(
                  matrixstore.forward_plan(k, n, rw, cfg.warps_per_cta), g.angles, n)),
             ("adjoint", t_ip, t_ix, t_v, g.num_voxels, g.num_rays,
              matrixstore.adjoint_plan(k, n, rw, cfg.warps_per_cta))]
    for kind, a, b, c, nr, nc, plan in sides:
        hf = matrixstore.build_format(a, b, c, nr, nc, plan, precision, 16, exp, budget,
                                      schedule=schedule)
        B, nk = pipeline.key_shape(g, kind)
        part = matrixstore.build_format_device(
            torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
            torch.from_numpy(c).to(dev), nr, nc, plan, precision, 16, exp, budget, schedule,
            B, nk, dev, exact=True)
        _compare(hf, part, precision)
        print(f"{kind} k={k} n={n} {precision} schedule={schedule}: device format == host "
              f"format ({hf.info['n_padded']} slab entries, {hf.info['n_groups']} groups)")


def _row_entries(T_or_arrays, info, precision, host):
    """Per (group, warp, row) the sorted nonzero slab entries (slot, value)."""
    warps, rpw = int(info["warps_per_cta"]), int(info["rows_per_warp"])
    if host:
        vals, slots = _host_words(T_or_arrays, precision)
        off, wid = T_or_arrays.arrays["slab_off"], T_or_arrays.arrays["slab_width"]
    else:
        T = {k: v.cpu().numpy() for k, v in T_or_arrays.tensors.items()}
        vals, slots = T["values"], T["slots"] if precision not in ("half", "mixed") else None
        off, wid = T["slab_off"], T["slab_width"]
    out = []
    for i in range(len(wid)):
        W = int(wid[i])
        if W == 0:
            continue
        blk = np.arange(W)[:, None] // 4 * rpw * 4 + np.arange(rpw)[None, :] * 4 + \
            (np.arange(W) % 4)[:, None]
        at = off[i] + blk                       # [step, row]
        for r in range(rpw):
            v = vals[at[:, r]]
            if slots is None:
                keep = (v.view(np.uint32) & 0xFFFF) != 0
                out.append(np.sort(v[keep].view(np.uint32)))
            else:
                keep = v != 0
                key = slots[at[:, r]][keep].astype(np.int64) * 2 ** 40 + \
                    np.argsort(np.argsort(v[keep]))
                out.append(np.sort(np.stack([slots[at[:, r]][keep].astype(np.float64),
                                             v[keep].astype(np.float64)], 1), axis=0))
    return out


@pytest.mark.parametrize("k,n,precision", [(180, 128, "mixed"), (64, 48, "single")])
def test_fast_schedule_places_the_same_entries(k, n, precision):
    """The default first-fit schedule: identical groups, maps and slab
    widths; every row holds the same entries in every slab, on other steps."""
    g = geometry.make_geometry(k, 1, n)
    A = geometry.build_system_matrix(g)
    ip, ix, v = A.host_csr32()
    cfg = pipeline.SystemConfig(precision=precision, ffactor=16, row_group=1)
    rw = pipeline._rows_per_warp(cfg)
    dev = geometry.device()
    exp = matrixstore.half_rescale_exponent(np.asarray(v)) if precision == "mixed" else 0
    plan = matrixstore.assign_forward_regimes(
        matrixstore.forward_plan(k, n, rw, cfg.warps_per_cta), g.angles, n)
    hf = matrixstore.build_format(ip, ix, v, g.num_rays, g.num_voxels, plan, precision, 16, exp,
                                  cfg.smem_budget_effective, schedule=True)
    part = matrixstore.build_format_device(
        torch.from_numpy(ip).to(dev), torch.from_numpy(ix).to(dev), torch.from_numpy(v).to(dev),
        g.num_rays, g.num_voxels, plan, precision, 16, exp, cfg.smem_budget_effective, True,
        n, n, dev)
    T = {k2: t.cpu().numpy() for k2, t in part.tensors.items()}
    for k2 in ("cta_group_ptr", "group_map_ptr", "group_map", "slab_off", "slab_width"):
        assert np.array_equal(T[k2][:len(hf.arrays[k2])], hf.arrays[k2]), k2
    a = _row_entries(hf, hf.info, precision, True)
    b = _row_entries(part, part.info, precision, False)
    assert len(a) == len(b)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_device_band_transpose_equals_host_transpose():
    g = geometry.make_geometry(64, 1, 48)
    A = geometry.build_system_matrix(g)
    ip, ix, v = A.host_csr32()
    t_ip, t_ix, t_v = pipeline._transpose(ip, ix, v, g.num_rays, g.num_voxels)
    dev = geometry.device()
    st = _lib.stream_handle(dev)
    n = g.grid_n
    for z0, z1 in ((0, 16), (16, 48)):
        lo, hi = z0 * n, z1 * n
        counts = torch.zeros(hi - lo, dtype=torch.int64, device=dev)
        chunks = [(0, 20), (20, 45), (45, 64)]
        csrs = [geometry.siddon_csr(g, k0, k1, dev) for k0, k1 in chunks]
        for (k0, k1), (c_ip, c_ix, _) in zip(chunks, csrs):
            _lib.call("xct_csr_col_counts", c_ip.data_ptr(), c_ix.data_ptr(), (k1 - k0) * n, lo,
                      hi, counts.data_ptr(), st)
        d_ip = torch.zeros(hi - lo + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts, 0, out=d_ip[1:])
        m = int(d_ip[-1])
        rows = torch.empty(m, dtype=torch.int32, device=dev)
        vals = torch.empty(m, dtype=torch.float64, device=dev)
        cur = torch.zeros(hi - lo, dtype=torch.int32, device=dev)
        prev = torch.zeros(hi - lo, dtype=torch.int32, device=dev)
        for (k0, k1), (c_ip, c_ix, c_v) in zip(chunks, csrs):
            _lib.call("xct_csr_transpose_band", c_ip.data_ptr(), c_ix.data_ptr(), c_v.data_ptr(),
                      (k1 - k0) * n, k0 * n, 7 * n, lo, hi, d_ip.data_ptr(), cur.data_ptr(),
                      prev.data_ptr(), rows.data_ptr(), vals.data_ptr(), st)
        want_ip = t_ip[lo:hi + 1] - t_ip[lo]
        assert np.array_equal(d_ip.cpu().numpy(), want_ip)
        assert np.array_equal(rows.cpu().numpy(), t_ix[t_ip[lo]:t_ip[hi]])
        assert np.array_equal(vals.cpu().numpy(), t_v[t_ip[lo]:t_ip[hi]])


@pytest.mark.parametrize("precision", ["mixed", "half"])
def test_streamed_device_build_equals_monolithic_host_build(precision, monkeypatch):
    """Whole operators: the streamed device build (chunks of views, bands of
    voxels) with the host's exact schedule gives the same projections, bit
    for bit, as the monolithic host build; with the default fast schedule
    the same to rounding."""
    g = geometry.make_geometry(96, 16, 64)
    monkeypatch.setenv("XCT_FMTD_EXACT", "1")
    monkeypatch.setenv("XCT_HOST_BUILD", "1")
    host = pipeline.assemble(g, pipeline.SystemConfig(precision=precision, ffactor=16,
                                                      build="monolithic"))
    monkeypatch.delenv("XCT_HOST_BUILD")
    monkeypatch.setattr(pipeline.StreamedAssembly, "CHUNK_NNZ", 2e5)    # several chunks
    monkeypatch.setattr(pipeline.StreamedAssembly, "BAND_NNZ_DEV", 3e5)  # several bands
    dev_sys = pipeline.assemble(g, pipeline.SystemConfig(precision=precision, ffactor=16,
                                                         build="streamed"))
    assert dev_sys.forward.blocks[0].hbm_bytes() > 0
    rng = np.random.default_rng(4)
    x = rng.random((g.num_voxels, 16)).astype(np.float32)
    y = rng.random((g.num_rays, 16)).astype(np.float32)
    assert np.array_equal(dev_sys.apply_forward(x)[0], host.apply_forward(x)[0])
    assert np.array_equal(dev_sys.apply_adjoint(y)[0], host.apply_adjoint(y)[0])
    # the streamed build records its non-empty rays / touched voxels, so its
    # exchange accounting equals the monolithic build's
    from dataclasses import asdict
    vd, vh = dev_sys.volume_reports(), host.volume_reports()
    assert all(asdict(vd[k]) == asdict(vh[k]) for k in ("projection", "backprojection"))
    monkeypatch.delenv("XCT_FMTD_EXACT")
    for mode in ("0", "adjoint", "all"):
        monkeypatch.setenv("XCT_FMTD_PAIRED", mode)
        fast = pipeline.assemble(g, pipeline.SystemConfig(precision=precision, ffactor=16,
                                                          build="streamed"))
        for a, b in ((fast.apply_forward(x)[0], host.apply_forward(x)[0]),
                     (fast.apply_adjoint(y)[0], host.apply_adjoint(y)[0])):
            rel = float(np.linalg.norm(a - b) / np.linalg.norm(b))
            print(f"{precision} paired={mode} schedule vs host: rel-L2 {rel:.2e}")
            assert rel <= (1e-3 if precision == "mixed" else 5e-3)


def _half_wavefronts(part, lanes_per_row=1):
    """LDS.128 wavefronts per half-warp step under the measured rule
    (tools/smem_share_bench.cu): one when each quarter reads <= 4 distinct
    records and the half's distinct records sit in distinct bank classes,
    else per quarter the worst class multiplicity.  Returns (wavefronts,
    half-steps) over all slabs of a packed (half/mixed) format."""
    T = {k: v.cpu().numpy() for k, v in part.tensors.items()}
    rpw = int(part.info["rows_per_warp"])
    slot = (T["values"].view(np.uint32) >> 20).astype(np.int64)
    wf = hs = 0
    for off, W in zip(T["slab_off"], T["slab_width"]):
        if W == 0:
            continue
        st = np.arange(W)
        at = off + (st[:, None] // 4) * rpw * 4 + np.arange(rpw)[None, :] * 4 + (st % 4)[:, None]
        s = slot[at]                                   # [W, rpw]
        for h in range(rpw // 16):
            for n in range(W):
                q0, q1 = set(s[n, 16 * h:16 * h + 8]), set(s[n, 16 * h + 8:16 * h + 16])
                u = q0 | q1
                if len(q0) <= 4 and len(q1) <= 4 and len({x & 7 for x in u}) == len(u):
                    wf += 1
                else:
                    for q in (q0, q1):
                        wf += max(sum(1 for x in q if x & 7 == c) for c in range(8))
                hs += 1
    return wf, hs


@pytest.mark.parametrize("mode", ["min", "fill", "greedy"])
@pytest.mark.parametrize("kind", ["forward", "adjoint"])
def test_paired_schedule_places_the_same_entries_and_merges(kind, mode, monkeypatch):
    """Sched mode 3 (paired half-warp schedule): the same groups, maps,
    widths and per-row slab entries as the host builder, fewer modelled
    LDS wavefronts than the default schedule (K6 results: the streamed
    test below)."""
    k, n, precision = 180, 128, "mixed"
    monkeypatch.setenv("XCT_FMTD_PAIRED", "all")          # view-paired forward lanes
    g = geometry.make_geometry(k, 1, n)
    A = geometry.build_system_matrix(g)
    ip, ix, v = A.host_csr32()
    cfg = pipeline.SystemConfig(precision=precision, ffactor=16, row_group=1)
    rw = pipeline._rows_per_warp(cfg)
    dev = geometry.device()
    exp = matrixstore.half_rescale_exponent(np.asarray(v))
    budget = cfg.smem_budget_effective
    if kind == "forward":
        a, b, c, nr, nc = ip, ix, v, g.num_rays, g.num_voxels
        plan = matrixstore.assign_forward_regimes(
            matrixstore.forward_plan(k, n, rw, cfg.warps_per_cta), g.angles, n)
    else:
        a, b, c = pipeline._transpose(ip, ix, v, g.num_rays, g.num_voxels)
        nr, nc = g.num_voxels, g.num_rays
        plan = matrixstore.adjoint_plan(k, n, rw, cfg.warps_per_cta)
    hf = matrixstore.build_format(a, b, c, nr, nc, plan, precision, 16, exp, budget, schedule=True)
    B, nk = pipeline.key_shape(g, kind)
    args = (torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), torch.from_numpy(c).to(dev),
            nr, nc, plan, precision, 16, exp, budget, True, B, nk, dev)
    monkeypatch.setenv("XCT_FMTD_PAIRED", "0")
    default = matrixstore.build_format_device(*args)
    monkeypatch.setenv("XCT_FMTD_PAIRED", "all")
    if mode == "fill":
        monkeypatch.setenv("XCT_FMTD_PAIRED_FILL", "1")
    if mode == "greedy":                     # first-fit colourings on both sides
        monkeypatch.setenv("XCT_FMTD_PAIRED_GREEDY", "1")
    paired = matrixstore.build_format_device(*args)
    T = {k2: t.cpu().numpy() for k2, t in paired.tensors.items()}
    for k2 in ("cta_group_ptr", "group_map_ptr", "group_map", "slab_off", "slab_width"):
        assert np.array_equal(T[k2][:len(hf.arrays[k2])], hf.arrays[k2]), k2
    ea = _row_entries(hf, hf.info, precision, True)
    eb = _row_entries(paired, paired.info, precision, False)
    assert len(ea) == len(eb)
    assert all(np.array_equal(x, y) for x, y in zip(ea, eb))
    assert paired.info["paired_half_steps"] > 0
    wf_d, hs = _half_wavefronts(default)
    wf_p, hs2 = _half_wavefronts(paired)
    assert hs == hs2
    print(f"{kind} mode {mode}: merged {paired.info['paired_merged_steps']} of "
          f"{paired.info['paired_half_steps']} half-steps; modelled LDS wavefronts per "
          f"half-step {wf_d / hs:.3f} (default) -> {wf_p / hs:.3f} (paired)")
    assert wf_p < wf_d
