"""Worker for tests/test_exchange_cpu.py (one process per rank, gloo): the
native domain partition's exchanges (domain.py) run with torch.distributed
p2p on CPU tensors -- owner-ordered footprints, in-place sends of
contiguous row slices, owner-first-then-senders-ascending accumulation, and
the adjoint's input gather -- on a real Siddon operator split by
equal-nnz tomogram cuts.  Writes this rank's owned results and footprint."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import xct_oracle as O  # noqa: E402
from paper_2009_07226_b200 import domain, hilbert  # noqa: E402


def main(out):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k, n, F = 40, 24, 3
    g = O.make_geom(k, 1, n)
    A = O.system_matrix(g)
    counts = np.bincount(A.indices, minlength=g.num_voxels)
    tomo = hilbert.decompose_weighted(hilbert.TileGrid("tomogram", n, n, 8), world, counts)
    sino = hilbert.decompose(hilbert.TileGrid("sinogram", k, n, 8), world)
    owner = np.empty(g.num_rays, np.int64)
    for q, s in enumerate(sino):
        owner[s.elements] = q
    cols = tomo[rank].elements
    rows_of = np.repeat(np.arange(g.num_rays), np.diff(A.indptr))
    mine = np.isin(A.indices, cols)
    fp = np.unique(rows_of[mine])
    order = np.argsort(owner[fp], kind="stable")
    fp = fp[order]
    seg = np.searchsorted(owner[fp], np.arange(world + 1))
    box = [None] * world
    dist.all_gather_object(box, (fp, seg))
    fp_of, seg_of = [b[0] for b in box], [b[1] for b in box]
    own_rows = sino[rank].elements
    L = domain.exchange_lists(fp_of, seg_of, own_rows, rank)
    rng = np.random.default_rng(7)
    x = rng.random((g.num_voxels, F)).astype(np.float32)
    y = rng.random((g.num_rays, F)).astype(np.float32)
    # forward: this rank's partials over its footprint (f32, entry order)
    pos = np.full(g.num_rays, -1)
    pos[fp] = np.arange(len(fp))
    part = np.zeros((len(fp), F), np.float32)
    for j in np.nonzero(mine)[0]:
        r = rows_of[j]
        part[pos[r]] += np.float32(A.values[j]) * x[A.indices[j]]
    ops, recvs = [], {}
    t = torch.from_numpy(part)
    for q in range(world):
        a, b = seg[q], seg[q + 1]
        if q != rank and b > a:
            ops.append(dist.P2POp(dist.isend, t[a:b].contiguous(), q))
    for s, p in L["recv_pos"].items():
        recvs[s] = torch.empty((len(p), F), dtype=torch.float32)
        ops.append(dist.P2POp(dist.irecv, recvs[s], s))
    for w in dist.batch_isend_irecv(ops) if ops else []:
        w.wait()
    o = np.zeros((len(own_rows), F), np.float32)
    a, b = seg[rank], seg[rank + 1]
    o[L["self_pos"]] += part[a:b]                     # owner first
    for s in sorted(recvs):                           # then senders ascending
        o[L["recv_pos"][s]] += recvs[s].numpy()
    # adjoint: gather y on the footprint from the owners, then local product
    yown = y[own_rows]
    xfp = np.zeros((len(fp), F), np.float32)
    xfp[a:b] = yown[L["self_pos"]]
    ops = [dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(yown[idx])), q)
           for q, idx in L["send_idx"].items()]
    rb = {}
    for s in range(world):
        a2, b2 = seg[s], seg[s + 1]
        if s != rank and b2 > a2:
            rb[s] = torch.empty((b2 - a2, F), dtype=torch.float32)
            ops.append(dist.P2POp(dist.irecv, rb[s], s))
    for w in dist.batch_isend_irecv(ops) if ops else []:
        w.wait()
    for s, buf in rb.items():
        xfp[seg[s]:seg[s + 1]] = buf.numpy()
    assert np.array_equal(xfp, y[fp])                  # the gather is exact
    cpos = np.full(g.num_voxels, -1)
    cpos[cols] = np.arange(len(cols))
    xo = np.zeros((len(cols), F), np.float64)
    for j in np.nonzero(mine)[0]:
        xo[cpos[A.indices[j]]] += A.values[j] * xfp[pos[rows_of[j]]]
    np.savez(out, rank=rank, own_rows=own_rows, o=o, cols=cols, xo=xo, fp=fp, part=part)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
