"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (the reference does not exist on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes ``tests/golden/*.npz`` (+ ``manifest.json``).  The fixtures pin the
CPU oracle (``oracle/xct_oracle.py``) and, through hashes of full-size
arrays, the GPU product path at config 1 (128x128, 180 angles, 16 slices).
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from xct import engine, geometry, hilbert, matrixstore, pipeline, solver  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_case(name, k, m, n, a0=0.0, a1=math.pi, vox=1.0, full=True):
    g = geometry.make_geometry(k, m, n, a0, a1, voxel_size=vox)
    A = geometry.build_system_matrix(g)
    rec = dict(k=k, m=m, n=n, a0=a0, a1=a1, vox=vox, nnz=A.nnz,
               sha_indptr=sha(A.indptr.astype(np.int64)),
               sha_indices=sha(A.indices.astype(np.int64)),
               sha_values=sha(A.values.astype(np.float64)))
    arrays = {}
    if full:
        arrays = dict(indptr=A.indptr, indices=A.indices, values=A.values)
    else:
        pick = np.unique(np.linspace(0, A.num_rows - 1, 64).astype(np.int64))
        arrays["sample_rows"] = pick
        for r in pick:
            s, e = A.indptr[r], A.indptr[r + 1]
            arrays[f"row{r}_idx"] = A.indices[s:e]
            arrays[f"row{r}_val"] = A.values[s:e]
    np.savez_compressed(OUT / f"csr_{name}.npz", **arrays)
    return rec, g, A


def main():
    manifest = {"csr": {}, "hilbert": {}, "engine": {}, "pipeline": {}, "cgls": {}}

    # ---- Siddon / system matrix --------------------------------------------------
    cases = [("g4x8", 4, 1, 8), ("g48x32", 48, 1, 32), ("g96x64", 96, 1, 64),
             ("g12x16", 12, 1, 16)]
    for name, k, m, n in cases:
        manifest["csr"][name], _, _ = csr_case(name, k, m, n)
    manifest["csr"]["two_voxel"], _, _ = csr_case("two_voxel", 1, 1, 2, vox=2.0)
    manifest["csr"]["odd_range"], _, _ = csr_case("odd_range", 7, 1, 13, 0.3, 2.9)
    manifest["csr"]["vox07"], _, _ = csr_case("vox07", 5, 1, 10, 0.0, math.pi / 3, vox=0.7)
    manifest["csr"]["n1"], _, _ = csr_case("n1", 3, 1, 1)
    rec, g1, A1 = csr_case("c1", 180, 16, 128, full=False)
    manifest["csr"]["c1"] = rec
    # angle-subset identity used by the CPU baseline extrapolation
    manifest["csr"]["c1_sub16"], _, _ = csr_case("c1_sub16", 16, 1, 128, 0.0,
                                                   16 * math.pi / 180, full=False)

    # ---- Hilbert ----------------------------------------------------------------
    hil = {}
    for tx, tz in [(1, 1), (2, 2), (4, 4), (3, 2), (5, 7), (16, 16), (23, 9), (6, 16)]:
        hil[f"order_{tx}x{tz}"] = np.array(hilbert.pseudo_hilbert_order(tx, tz), np.int64)
    hil["d2xy_o3"] = np.array([hilbert.hilbert_d2xy(3, d) for d in range(64)], np.int64)
    for (r, c, t, p) in [(64, 64, 8, 4), (32, 32, 8, 3), (48, 32, 8, 4), (180, 128, 8, 8),
                         (128, 128, 8, 8), (90, 64, 8, 6), (37, 29, 5, 7)]:
        grid = hilbert.TileGrid("tomogram", r, c, t)
        subs = hilbert.decompose(grid, p)
        key = f"dec_{r}x{c}_t{t}_p{p}"
        hil[key + "_sizes"] = np.array([s.num_elements for s in subs], np.int64)
        hil[key + "_elems"] = np.concatenate([s.elements for s in subs])
    grid = hilbert.TileGrid("sinogram", 13, 11, 4)
    hil["tile_elems_13x11_t4"] = np.concatenate(
        [grid.tile_elements(x, z) for z in range(grid.tiles_z) for x in range(grid.tiles_x)])
    np.savez_compressed(OUT / "hilbert.npz", **hil)

    # ---- engine: staged projection per precision --------------------------------
    g32 = geometry.make_geometry(48, 1, 32)
    A32 = geometry.build_system_matrix(g32)
    blk = matrixstore.block_from_matrix(A32)
    blkT = matrixstore.transpose(blk)
    eng = {}
    rng = np.random.default_rng(42)
    for ff in (1, 4, 16):
        X = rng.random((blk.num_cols, ff))
        Yin = rng.random((blk.num_rows, ff))
        eng[f"X_f{ff}"] = X
        eng[f"Y_f{ff}"] = Yin
        for prec in ("double", "single", "mixed", "half"):
            for cap in (96 * 1024, 4 * 1024, None):
                ctag = "none" if cap is None else str(cap)
                st = matrixstore.build_staged(blk, cap, 4, ff, precision=prec)
                out = engine.project(st, engine.Minibatch.from_columns(X, prec)).values
                eng[f"fwd_{prec}_f{ff}_c{ctag}"] = out
                stT = matrixstore.build_staged(blkT, cap, 4, ff, precision=prec)
                outT = engine.project(stT, engine.Minibatch.from_columns(Yin, prec)).values
                eng[f"adj_{prec}_f{ff}_c{ctag}"] = outT
    eng["exp_g32_mixed"] = np.array(matrixstore.half_rescale_exponent(A32.values))
    np.savez_compressed(OUT / "engine_g32.npz", **eng)

    # ---- pipeline: full operator application ------------------------------------
    pip = {}
    g64 = geometry.make_geometry(96, 1, 64)
    A64 = geometry.build_system_matrix(g64)
    x64 = geometry.generate_phantom("shepp-logan-like", 64, 5).slices_as_columns()
    rng = np.random.default_rng(7)
    y64 = rng.random((A64.num_rows, 5)).astype(np.float32)
    pip["x64"], pip["y64"] = x64, y64
    for prec in ("double", "single", "mixed", "half"):
        for ff in (4, 16):
            sysm = pipeline.assemble(g64, pipeline.SystemConfig(precision=prec, ffactor=ff))
            f, st = sysm.apply_forward(x64.astype(np.float32))
            a, _ = sysm.apply_adjoint(y64)
            pip[f"g64_fwd_{prec}_f{ff}"] = f
            pip[f"g64_adj_{prec}_f{ff}"] = a
            pip[f"g64_fwdfac_{prec}_f{ff}"] = np.array([s.factor for s in st])
    # data-parallel partitions (Hilbert subdomains), direct plan
    for prec in ("double", "single"):
        for p_d in (4, 6):
            sysm = pipeline.assemble(g64, pipeline.SystemConfig(
                precision=prec, ffactor=4, p_d=p_d, comm_strategy="direct"))
            f, _ = sysm.apply_forward(x64.astype(np.float32))
            a, _ = sysm.apply_adjoint(y64)
            pip[f"g64_pd{p_d}_fwd_{prec}"] = f
            pip[f"g64_pd{p_d}_adj_{prec}"] = a
    np.savez_compressed(OUT / "pipeline_g64.npz", **pip)

    # c1 operator outputs: hashed (full arrays are too large to commit)
    ph1 = geometry.generate_phantom("shepp-logan-like", 128, 16)
    x1 = ph1.slices_as_columns().astype(np.float32)
    sino1 = geometry.simulate_measurements(A1, ph1, 0.0, 0)
    y1 = sino1.slices_as_columns()
    manifest["pipeline"]["c1_y_sha"] = sha(y1.astype(np.float64))
    c1 = {"y_sample": y1[::97]}
    for prec in ("single", "mixed"):
        sysm = pipeline.assemble(g1, pipeline.SystemConfig(precision=prec, ffactor=16))
        f, _ = sysm.apply_forward(x1)
        a, _ = sysm.apply_adjoint(y1.astype(np.float32))
        manifest["pipeline"][f"c1_fwd_{prec}_sha"] = sha(f)
        manifest["pipeline"][f"c1_adj_{prec}_sha"] = sha(a)
        c1[f"fwd_{prec}_sample"] = f[::97]
        c1[f"adj_{prec}_sample"] = a[::61]
        res = solver.cgls_solve(sysm, y1, solver.SolveConfig(max_iters=30, precision=prec))
        manifest["cgls"][f"c1_{prec}_x_sha"] = sha(res.x)
        c1[f"cg_{prec}_x_sample"] = res.x[::61]
        c1[f"cg_{prec}_residual"] = np.array(res.residual_history)
        c1[f"cg_{prec}_gradient"] = np.array(res.gradient_history)
        c1[f"cg_{prec}_x"] = res.x.astype(np.float32)
        print("c1", prec, "done", flush=True)
    np.savez_compressed(OUT / "c1.npz", **c1)

    # ---- CGLS on the solver test problem ----------------------------------------
    g90 = geometry.make_geometry(90, 1, 64)
    A90 = geometry.build_system_matrix(g90)
    disk = geometry.generate_phantom("uniform-disk", 64, 3)
    y90 = geometry.simulate_measurements(A90, disk, 0.01, 3).slices_as_columns()
    cg = {"y90": y90}
    for prec in ("double", "single", "mixed", "half"):
        sysm = pipeline.assemble(g90, pipeline.SystemConfig(precision=prec, ffactor=4))
        res = solver.cgls_solve(sysm, y90, solver.SolveConfig(max_iters=12, precision=prec))
        cg[f"{prec}_x"] = res.x
        cg[f"{prec}_residual"] = np.array(res.residual_history)
        cg[f"{prec}_gradient"] = np.array(res.gradient_history)
        cg[f"{prec}_counts"] = np.array([res.projections, res.backprojections])
    np.savez_compressed(OUT / "cgls_g90.npz", **cg)

    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True))
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
