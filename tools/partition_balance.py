#!/usr/bin/env python
"""Per-rank SpMM work of the image-domain partition at a full-size geometry
(GPU: entries per voxel and per ray from the device Siddon, K1/K2 + K4
counts).  For P in {2, 4, 8}: max/mean of the nnz each rank's SpMM covers,
for the reference's equal-tile-count Hilbert cuts (src/hilbert.py:181-200)
and for cuts at equal cumulative nnz (hilbert.decompose_weighted):

  forward  A[:, T_r]         weights = entries per voxel (column nnz)
  adjoint  A[G_r, :]^T       weights = entries per ray   (reference scheme)
  adjoint  A[:, T_r]^T       = the forward block transposed (this build)

  python tools/partition_balance.py 2048 2048 > profiles/r02_partition_balance_c5.json
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2009_07226_b200 import _lib, geometry, hilbert  # noqa: E402


def main(n, k, tile=8):
    g = geometry.make_geometry(k, 1, n)
    dev = geometry.device()
    st = _lib.stream_handle(dev)
    col = torch.zeros(g.num_voxels, dtype=torch.int64, device=dev)
    row = np.zeros(g.num_rays, np.int64)
    per = max(1, int(4e8 // (1.2 * n * n)))
    for k0 in range(0, k, per):
        k1 = min(k, k0 + per)
        ip, ix, _ = geometry.siddon_csr(g, k0, k1, dev)
        _lib.call("xct_csr_col_counts", ip.data_ptr(), ix.data_ptr(), (k1 - k0) * n, 0,
                  g.num_voxels, col.data_ptr(), st)
        row[k0 * n:k1 * n] = torch.diff(ip).cpu().numpy()
        del ip, ix
    col = col.cpu().numpy().astype(np.float64)
    tomo = hilbert.TileGrid("tomogram", n, n, tile)
    sino = hilbert.TileGrid("sinogram", k, n, tile)
    out = {"n": n, "k": k, "nnz": int(row.sum()), "tile": tile, "parts": {}}
    for P in (2, 4, 8):
        r = {}
        for name, grid, w in (("forward (tomogram tiles, column nnz)", tomo, col),
                              ("adjoint reference (sinogram tiles, row nnz)", sino, row)):
            for cut, parts in (("equal tiles", hilbert.decompose(grid, P)),
                               ("equal nnz", hilbert.decompose_weighted(grid, P, w))):
                loads = np.array([w[s.elements].sum() for s in parts])
                r[f"{name}, {cut}"] = {"max_over_mean": float(loads.max() / loads.mean()),
                                       "max_over_min": float(loads.max() / loads.min())}
        out["parts"][P] = r
        print(P, json.dumps(r), file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
