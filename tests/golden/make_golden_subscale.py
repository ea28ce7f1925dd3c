"""Sub-scale parity fixtures made by running the REFERENCE:
N = K = 256 (30 CGLS iterations, single and mixed) and N = K = 512 (5
iterations), plus the reference's own stage-capacity noise floor at 256.

Run in the build container only (the reference does not exist on the GPU
box; each 256 job is ~3 min and ~3 GB, each 512 job ~12 min and ~22 GB):

    python tests/golden/make_golden_subscale.py [256|512|all]

Inputs are handed to the reference as float32 measurements (the reference
upcasts them to float64, src/solver.py:137), so the fixture's ``y`` is the
exact input of both implementations.

Writes ``tests/golden/sub256.npz`` / ``sub512.npz`` and
``tests/golden/sub_manifest.json`` (noise floors, timings, hashes).
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import sys
import time
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

# (stage_capacity_bytes, block_partitions): the reference default and the two
# alternative stagings whose spread is the reference's own order noise floor
STAGINGS = {"default": (96 * 1024, 4), "unstaged": (None, 1), "small": (4096, 8)}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def problem(n: int):
    """256: random-blobs (distinct slices, seed 0); 512: Shepp-Logan (every
    slice identical, src/geometry.py:337-339 -- the fixture keeps one column);
    128: config 1 itself (180 views, Shepp-Logan, float64 y)."""
    from xct import geometry
    g = geometry.make_geometry(180 if n == 128 else n, 16, n)
    A = geometry.build_system_matrix(g)
    if n == 128:
        vol = geometry.generate_phantom("shepp-logan-like", n, 16)
        y = geometry.simulate_measurements(A, vol, 0.0, 0).slices_as_columns()
        return g, y, vol.slices_as_columns()
    kind = "random-blobs" if n == 256 else "shepp-logan-like"
    vol = geometry.generate_phantom(kind, n, 16, seed=0)
    y = geometry.simulate_measurements(A, vol, 0.0, 0).slices_as_columns()
    return g, y.astype(np.float32), vol.slices_as_columns()   # noqa


def job(args):
    n, prec, staging, iters = args
    from xct import pipeline, solver
    t0 = time.perf_counter()
    g, y32, _ = problem(n)
    cap, parts = STAGINGS[staging]
    sysm = pipeline.assemble(g, pipeline.SystemConfig(precision=prec, ffactor=16,
                                                      stage_capacity_bytes=cap,
                                                      block_partitions=parts))
    t1 = time.perf_counter()
    res = solver.cgls_solve(sysm, y32, solver.SolveConfig(max_iters=iters, precision=prec))
    t2 = time.perf_counter()
    print(f"n={n} {prec} {staging}: assemble {t1 - t0:.1f} s, cgls {t2 - t1:.1f} s", flush=True)
    return dict(n=n, prec=prec, staging=staging, iters=iters, x=res.x.astype(np.float32),
                x_sha=sha(res.x), residual=np.array(res.residual_history),
                gradient=np.array(res.gradient_history), assemble_s=t1 - t0, cgls_s=t2 - t1)


def main(which: str = "all"):
    man_path = OUT / "sub_manifest.json"
    manifest = json.loads(man_path.read_text()) if man_path.exists() else {}
    jobs = []
    if which in ("256", "all"):
        jobs += [(256, p, s, 30) for p in ("single", "mixed") for s in STAGINGS]
    if which in ("512", "all"):
        jobs += [(512, p, "default", 5) for p in ("single", "mixed")]
    if which in ("128", "all"):          # config 1: the reference's own floor only
        jobs += [(128, p, s, 30) for p in ("single", "mixed") for s in STAGINGS]
    procs = 6 if which in ("256", "128") else 2
    with mp.get_context("fork").Pool(min(procs, len(jobs)), maxtasksperchild=1) as pool:
        runs = pool.map(job, jobs, chunksize=1)
    for n in sorted({r["n"] for r in runs}):
        _, y32, _ = problem(n)
        arrays, rec = {}, {"iters": None, "floor": {}}
        one_col = n == 512
        keep_arrays = n != 128           # c1's arrays are in tests/golden/c1.npz
        arrays["y"] = y32[:, 0] if one_col else y32
        rec["y_sha"] = sha(y32)
        rec["phantom"] = "random-blobs seed 0" if n == 256 else "shepp-logan-like"
        for r in (r for r in runs if r["n"] == n):
            key = f"{r['prec']}_{r['staging']}"
            rec["iters"] = r["iters"]
            rec[f"{key}_x_sha"] = r["x_sha"]
            rec[f"{key}_assemble_s"] = r["assemble_s"]
            rec[f"{key}_cgls_s"] = r["cgls_s"]
            if r["staging"] == "default":
                arrays[f"{r['prec']}_x"] = r["x"][:, 0] if one_col else r["x"]
                arrays[f"{r['prec']}_residual"] = r["residual"]
                arrays[f"{r['prec']}_gradient"] = r["gradient"]
        # the reference against itself with only the staging changed
        for prec in ("single", "mixed"):
            base = next((r for r in runs if r["n"] == n and r["prec"] == prec
                         and r["staging"] == "default"), None)
            alts = [r for r in runs if r["n"] == n and r["prec"] == prec
                    and r["staging"] != "default"]
            if base is None or not alts:
                continue
            xb = base["x"].astype(np.float64)
            rec["floor"][prec] = {
                r["staging"]: {
                    "x_rel_l2": float(np.linalg.norm(r["x"] - xb) / np.linalg.norm(xb)),
                    "curve_max_rel": float(np.max(np.abs(r["residual"] / base["residual"] - 1))),
                } for r in alts}
        manifest[f"sub{n}"] = rec
        if keep_arrays:
            np.savez_compressed(OUT / f"sub{n}.npz", **arrays)
        print(f"sub{n}: floor {json.dumps(rec['floor'])}", flush=True)
    man_path.write_text(json.dumps(manifest, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
