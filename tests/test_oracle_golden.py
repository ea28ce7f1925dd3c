"""Pin the CPU oracle to the reference's own outputs (golden vectors made by
``tests/golden/make_golden.py`` from /root/reference).  CPU only."""

import hashlib
import math

import numpy as np
import pytest

from conftest import load_golden
import xct_oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CSR_CASES = ["g4x8", "g48x32", "g96x64", "g12x16", "two_voxel", "odd_range", "vox07", "n1"]


@pytest.mark.parametrize("name", CSR_CASES)
def test_siddon_csr_bit_exact(golden_manifest, name):
    rec = golden_manifest["csr"][name]
    g = O.make_geom(rec["k"], rec["m"], rec["n"], rec["a0"], rec["a1"], rec["vox"])
    A = O.system_matrix(g)
    gold = load_golden(f"csr_{name}")
    assert np.array_equal(A.indptr, gold["indptr"])
    assert np.array_equal(A.indices, gold["indices"])
    assert np.array_equal(A.values, gold["values"])  # float64 bit-exact
    assert sha(A.values) == rec["sha_values"]


def test_siddon_c1_hashes(golden_manifest):
    rec = golden_manifest["csr"]["c1"]
    A = O.system_matrix(O.make_geom(180, 16, 128))
    assert A.nnz == rec["nnz"] == 3524296
    assert sha(A.indptr.astype(np.int64)) == rec["sha_indptr"]
    assert sha(A.indices.astype(np.int64)) == rec["sha_indices"]
    assert sha(A.values) == rec["sha_values"]


def test_hilbert_orders_and_decompositions():
    gold = load_golden("hilbert")
    for key in gold.files:
        if key.startswith("order_"):
            tx, tz = map(int, key[6:].split("x"))
            assert np.array_equal(np.array(O.pseudo_order(tx, tz)), gold[key])
    assert np.array_equal(np.array([O.h_d2xy(3, d) for d in range(64)]), gold["d2xy_o3"])
    for key in gold.files:
        if key.startswith("dec_") and key.endswith("_sizes"):
            body = key[4:-6]
            shape, t, p = body.split("_")
            r, c = map(int, shape.split("x"))
            subs = O.decompose(r, c, int(t[1:]), int(p[1:]))
            assert np.array_equal([len(s) for s in subs], gold[key])
            assert np.array_equal(np.concatenate(subs), gold[key[:-6] + "_elems"])
    cells = [O.tile_cells(13, 11, 4, x, z) for z in range(4) for x in range(3)]
    assert np.array_equal(np.concatenate(cells), gold["tile_elems_13x11_t4"])


def test_staged_projection_bit_exact_all_precisions():
    gold = load_golden("engine_g32")
    g = O.make_geom(48, 1, 32)
    A = O.system_matrix(g)
    blk = O.whole_block(A)
    blkT = O.transpose_block(blk)
    assert O.rescale_exp(A.values) == int(gold["exp_g32_mixed"])
    for ff in (1, 4, 16):
        X, Y = gold[f"X_f{ff}"], gold[f"Y_f{ff}"]
        for prec in ("double", "single", "mixed", "half"):
            e = O.rescale_exp(blk.values) if prec in ("half", "mixed") else 0
            eT = O.rescale_exp(blkT.values) if prec in ("half", "mixed") else 0
            for cap, tag in ((96 * 1024, "98304"), (4 * 1024, "4096"), (None, "none")):
                out = O.staged_apply(blk, X.astype(O.STORE[prec]), prec, e, cap, 4)
                assert np.array_equal(out, gold[f"fwd_{prec}_f{ff}_c{tag}"]), (prec, ff, tag)
                outT = O.staged_apply(blkT, Y.astype(O.STORE[prec]), prec, eT, cap, 4)
                assert np.array_equal(outT, gold[f"adj_{prec}_f{ff}_c{tag}"]), (prec, ff, tag)


def test_operator_application_bit_exact():
    gold = load_golden("pipeline_g64")
    g = O.make_geom(96, 1, 64)
    A = O.system_matrix(g)
    x, y = gold["x64"].astype(np.float32), gold["y64"]
    for prec in ("double", "single", "mixed", "half"):
        for ff in (4, 16):
            op = O.Operator(A, g, prec, ff)
            f, fac = op.forward(x)
            a, _ = op.adjoint(y)
            assert np.array_equal(f, gold[f"g64_fwd_{prec}_f{ff}"]), (prec, ff)
            assert np.array_equal(a, gold[f"g64_adj_{prec}_f{ff}"]), (prec, ff)
            assert np.array_equal(fac, gold[f"g64_fwdfac_{prec}_f{ff}"])


def test_partitioned_operator_matches_reference_direct_plan():
    gold = load_golden("pipeline_g64")
    g = O.make_geom(96, 1, 64)
    A = O.system_matrix(g)
    x, y = gold["x64"].astype(np.float32), gold["y64"]
    for prec in ("double", "single"):
        for p_d in (4, 6):
            op = O.Operator(A, g, prec, 4, p_d=p_d)
            assert np.array_equal(op.forward(x)[0], gold[f"g64_pd{p_d}_fwd_{prec}"])
            assert np.array_equal(op.adjoint(y)[0], gold[f"g64_pd{p_d}_adj_{prec}"])


def test_cgls_histories_match_reference():
    gold = load_golden("cgls_g90")
    g = O.make_geom(90, 1, 64)
    A = O.system_matrix(g)
    y = gold["y90"]
    for prec in ("double", "single", "mixed", "half"):
        op = O.Operator(A, g, prec, 4)
        res = O.cgls(op, y, 12, prec)
        assert [res["projections"], res["backprojections"]] == list(gold[f"{prec}_counts"])
        # same BLAS vdot order as the reference => bit-identical
        assert np.array_equal(res["x"], gold[f"{prec}_x"]), prec
        assert np.array_equal(res["residual"], gold[f"{prec}_residual"])
        assert np.array_equal(res["gradient"], gold[f"{prec}_gradient"])


def test_c1_operator_and_cgls(golden_manifest):
    """Config 1 end to end: y, forward/adjoint and 30-iteration CGLS."""
    gold = load_golden("c1")
    g = O.make_geom(180, 16, 128)
    A = O.system_matrix(g)
    vol = O.phantom("shepp-logan-like", 128, 16)
    y = O.measure(A, vol)
    assert sha(y) == golden_manifest["pipeline"]["c1_y_sha"]
    x = vol.reshape(16, -1).T.astype(np.float32)
    for prec in ("single", "mixed"):
        op = O.Operator(A, g, prec, 16)
        f, _ = op.forward(x)
        a, _ = op.adjoint(y.astype(np.float32))
        assert sha(f) == golden_manifest["pipeline"][f"c1_fwd_{prec}_sha"]
        assert sha(a) == golden_manifest["pipeline"][f"c1_adj_{prec}_sha"]
        res = O.cgls(op, y, 30, prec)
        assert np.array_equal(res["residual"], gold[f"cg_{prec}_residual"])
        assert sha(res["x"]) == golden_manifest["cgls"][f"c1_{prec}_x_sha"]


def test_slice_groups_rule():
    assert O.slice_groups(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert O.slice_groups(2, 4) == [(0, 1), (1, 2)]


def test_double_cgls_order_noise_floor():
    """Pins the tolerance of the GPU double-mode CGLS test: an exactly
    rounded dot (math.fsum) instead of numpy's vdot moves x by ~1.3e-5 on the
    noisy g90 problem after 12 iterations (single/mixed/half: 0)."""
    gold = load_golden("cgls_g90")
    g = O.make_geom(90, 1, 64)
    op = O.Operator(O.system_matrix(g), g, "double", 4)
    orig = O._vdot
    try:
        O._vdot = lambda a, b: math.fsum((a.astype(np.float64) * b.astype(np.float64)).ravel())
        r = O.cgls(op, gold["y90"], 12, "double")
    finally:
        O._vdot = orig
    d = np.linalg.norm(r["x"] - gold["double_x"]) / np.linalg.norm(gold["double_x"])
    assert 1e-6 < d < 3e-5
