#!/usr/bin/env python
"""Union/sum ratio of neighbouring rows' column sets of the Siddon operator
(the saving of K6's grouped rows): for A, units of adjacent views x
detectors; for A^T, units of adjacent voxels.  Uses the CPU oracle (test
infrastructure), so keep N, K <= 256.

  python tools/union_study.py 256 256
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import xct_oracle as O  # noqa: E402


def union_ratio(ptr, idx, groups):
    tot = uni = 0
    for grp in groups:
        cols = [idx[ptr[r]:ptr[r + 1]] for r in grp]
        tot += sum(len(c) for c in cols)
        uni += len(np.unique(np.concatenate(cols)))
    return uni / tot


def main(N, K):
    g = O.make_geom(K, 1, N)
    A = O.system_matrix(g)
    ip, ix = A.indptr, A.indices
    T = O.transpose_block(O.whole_block(A))
    rng = np.random.default_rng(0)
    vox = list(zip(rng.integers(0, N - 4, 400), rng.integers(0, N - 4, 400)))
    for name, offs in [("pair_x", [(0, 0), (0, 1)]), ("pair_z", [(0, 0), (1, 0)]),
                       ("quad 2x2", [(a, b) for a in range(2) for b in range(2)]),
                       ("2x4", [(a, b) for a in range(2) for b in range(4)])]:
        groups = [[(z + a) * N + x + b for a, b in offs] for z, x in vox]
        print(f"adjoint {name:9s} union/sum {union_ratio(T.indptr, T.indices, groups):.3f}")
    rays = list(zip(rng.integers(0, K - 4, 400), rng.integers(N // 8, N - N // 8 - 4, 400)))
    for name, offs in [("views2", [(0, 0), (1, 0)]), ("dets2", [(0, 0), (0, 1)]),
                       ("2x2", [(a, b) for a in range(2) for b in range(2)]),
                       ("4x2", [(a, b) for a in range(4) for b in range(2)])]:
        groups = [[(k + a) * N + c + b for a, b in offs] for k, c in rays]
        print(f"forward {name:9s} union/sum {union_ratio(ip, ix, groups):.3f}")


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
