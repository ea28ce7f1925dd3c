#!/usr/bin/env python
"""CPU timing of the K5 format builder on a Siddon matrix made by the test
oracle (tools only; cached under /tmp).  XCT_VERBOSE=1 prints phase times.

  python tools/build_bench.py --n 256 --angles 256 [--precision single]
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--angles", type=int, default=256)
    ap.add_argument("--precision", default="single")
    ap.add_argument("--side", default="both")
    args = ap.parse_args()
    from paper_2009_07226_b200 import matrixstore
    n, k = args.n, args.angles
    cache = Path(f"/tmp/xb/csr_{n}_{k}.npz")
    if cache.exists():
        z = np.load(cache)
        ip, ix, v = z["ip"], z["ix"], z["v"]
    else:
        from oracle import xct_oracle as O
        g = O.make_geom(k, 1, n)
        A = O.system_matrix(g)
        ip, ix, v = A.indptr, A.indices.astype(np.int32), A.values
        np.savez(cache, ip=ip, ix=ix, v=v)
    import math
    angles = [i * math.pi / k for i in range(k)]
    rw = 32 // matrixstore.lanes_for(16, args.precision, 2)
    if args.side in ("both", "forward"):
        plan = matrixstore.assign_forward_regimes(matrixstore.forward_plan(k, n, rw, 16), angles, n)
        t0 = time.perf_counter()
        hf = matrixstore.build_format(ip, ix, v, k * n, n * n, plan, args.precision, 16, 0,
                                      schedule=True)
        print(f"forward nnz {len(ix)} padded {int(hf.info['n_padded'])} "
              f"{time.perf_counter() - t0:.3f} s")
    if args.side in ("both", "adjoint"):
        from paper_2009_07226_b200.pipeline import _transpose
        t_ip, t_ix, t_v = _transpose(ip, ix, v, k * n, n * n)
        plan = matrixstore.adjoint_plan(k, n, rw, 16)
        t0 = time.perf_counter()
        hf = matrixstore.build_format(t_ip, t_ix, t_v, n * n, k * n, plan, args.precision, 16, 0,
                                      schedule=True)
        print(f"adjoint padded {int(hf.info['n_padded'])} {time.perf_counter() - t0:.3f} s")


if __name__ == "__main__":
    main()
