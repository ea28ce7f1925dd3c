"""Sub-scale parity of the DEFAULT (fast, native-order) path against the
reference run at N = K = 256 (30 CGLS iterations) and N = K = 512 (5
iterations), fixtures made by tests/golden/make_golden_subscale.py.

Tolerances follow SURVEY.md §8(c):
  * reference order ("reference" staging) reproduces the reference bit for
    bit: x sha256 equal;
  * native order, FP32: x within 2x the reference's OWN stage-capacity noise
    floor at that geometry (the reference against itself with only the
    staging changed, tests/golden/sub_manifest.json), residual curve within
    2x its curve floor;
  * native order, FP16 storage: residual curve within 2% per iteration or
    2x the reference's own curve floor, whichever is larger (the floor is
    2.7% at N = 256), and x within 2x the mixed noise floor;
  * <= 10 iterations (N = 512, 5 iterations): FP32 x within 1e-5.
Every test prints the deviation it measured.
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"


def _manifest():
    p = GOLD / "sub_manifest.json"
    return json.loads(p.read_text()) if p.exists() else {}


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _fixture(n):
    p = GOLD / f"sub{n}.npz"
    if not p.exists():
        pytest.skip(f"{p.name} not generated")
    return np.load(p), _manifest()[f"sub{n}"]


def _solve(n, y, prec, iters, **cfg):
    from paper_2009_07226_b200 import geometry, pipeline, solver
    g = geometry.make_geometry(n, y.shape[1], n)
    sysm = pipeline.assemble(g, pipeline.SystemConfig(precision=prec, ffactor=16, **cfg))
    res = solver.cgls_solve(sysm, y, solver.SolveConfig(max_iters=iters, precision=prec))
    geometry.clear_matrix_cache()
    return res, sysm


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("prec", ["single", "mixed"])
def test_sub256_reference_order_bit_exact(prec):
    gold, man = _fixture(256)
    res, _ = _solve(256, gold["y"], prec, man["iters"], order="reference")
    print(f"sub256 {prec} reference order: x sha {'==' if _sha(res.x) == man[f'{prec}_default_x_sha'] else '!='} reference")
    assert _sha(res.x) == man[f"{prec}_default_x_sha"]
    # the residual history's norms are f64 dots in another summation order
    np.testing.assert_allclose(res.residual_history, gold[f"{prec}_residual"], rtol=1e-12)


@pytest.mark.parametrize("prec", ["single", "mixed"])
def test_sub256_native_order_within_reference_noise_floor(prec):
    gold, man = _fixture(256)
    res, sysm = _solve(256, gold["y"], prec, man["iters"])
    blk = sysm.forward.blocks[0]
    floor = man["floor"][prec]
    x_floor = max(v["x_rel_l2"] for v in floor.values())
    c_floor = max(v["curve_max_rel"] for v in floor.values())
    x_dev = _rel(res.x, gold[f"{prec}_x"].astype(np.float64))
    curve = np.array(res.residual_history)
    c_dev = float(np.max(np.abs(curve / gold[f"{prec}_residual"] - 1.0)))
    print(f"sub256 {prec} native (row_group {blk.info.row_group}): x rel-L2 {x_dev:.3e} "
          f"(reference floor {x_floor:.3e}), residual curve max rel dev {c_dev:.3e} "
          f"(reference floor {c_floor:.3e})")
    assert len(curve) == man["iters"]
    assert x_dev <= 2.0 * x_floor
    # SURVEY §8(c) proposes 2% per iteration for FP16 storage; the
    # reference's own mixed curve moves by up to 2.7% at this geometry when
    # only its staging changes, so the bound is the larger of the two
    assert c_dev <= max(2.0 * c_floor, 0.02 if prec == "mixed" else 1e-6)


@pytest.mark.parametrize("prec", ["single", "mixed"])
def test_sub512_native_order(prec):
    gold, man = _fixture(512)
    y = np.repeat(gold["y"][:, None], 16, axis=1)        # identical slices
    res, _ = _solve(512, y, prec, man["iters"])
    x_dev = _rel(res.x[:, 0], gold[f"{prec}_x"].astype(np.float64))
    curve = np.array(res.residual_history)
    c_dev = float(np.max(np.abs(curve / gold[f"{prec}_residual"] - 1.0)))
    # every slice identical in, identical out
    same = bool(np.all(res.x == res.x[:, :1]))
    print(f"sub512 {prec} native, {man['iters']} iterations: x rel-L2 {x_dev:.3e}, "
          f"residual curve max rel dev {c_dev:.3e}, slices identical: {same}")
    assert same
    tol = 1e-5 if prec == "single" else 2e-3
    assert x_dev <= tol
    assert c_dev <= (1e-5 if prec == "single" else 0.02)


def test_sub512_reference_order_bit_exact():
    gold, man = _fixture(512)
    y = np.repeat(gold["y"][:, None], 16, axis=1)
    res, _ = _solve(512, y, "mixed", man["iters"], order="reference")
    x0 = res.x[:, 0].astype(np.float32)
    print("sub512 mixed reference order: x equal to the reference:",
          bool(np.array_equal(x0, gold["mixed_x"])))
    assert np.array_equal(x0, gold["mixed_x"])


def test_mixed_converges_to_single_plateau_sub256():
    """tests/test_solver.py:137-148 at N = K = 256 on the default path:
    FP16 storage tracks the FP32 curve to the same order of magnitude."""
    gold, man = _fixture(256)
    rel = {}
    for prec in ("single", "mixed"):
        res, _ = _solve(256, gold["y"], prec, 24)
        rel[prec] = res.residual_history[-1]
    print(f"sub256 iteration 24: single {rel['single']:.4e}, mixed {rel['mixed']:.4e}, "
          f"ratio {rel['mixed'] / rel['single']:.3f}")
    assert rel["mixed"] <= 3.0 * rel["single"]


def test_mixed_converges_to_single_plateau_problem64():
    """The reference's own case verbatim (tests/test_solver.py:22-28,
    :137-148): K = 90, N = 64 uniform disk, noiseless, F = 1, 24 iterations."""
    from paper_2009_07226_b200 import geometry, pipeline, solver
    g = geometry.make_geometry(90, 1, 64)
    A = geometry.build_system_matrix(g)
    y = geometry.simulate_measurements(A, geometry.generate_phantom("uniform-disk", 64, 1),
                                       0.0, 0).slices_as_columns()
    rel = {}
    for prec in ("single", "mixed"):
        sysm = pipeline.assemble(g, pipeline.SystemConfig(precision=prec, ffactor=1))
        rel[prec] = solver.cgls_solve(sysm, y, solver.SolveConfig(
            max_iters=24, precision=prec)).residual_history[-1]
    print(f"problem64 iteration 24: single {rel['single']:.4e}, mixed {rel['mixed']:.4e}")
    assert rel["mixed"] <= 3.0 * rel["single"]
