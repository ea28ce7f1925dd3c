"""Multi-process host logic on CPU (gloo, world_size 2): the slice-batch
rule and the broadcast of a staged operator side from the building rank."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import xct_oracle as O
from paper_2009_07226_b200 import parallel


def test_slice_groups_matches_reference_rule():
    assert parallel.slice_groups(10, 3) == O.slice_groups(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert parallel.slice_groups(2048, 8)[-1] == (1792, 2048)
    assert parallel.slice_groups(3, 8) == [(0, 1), (1, 2), (2, 3)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_broadcast_side_gloo_world2(tmp_path):
    port = _free_port()
    worker = Path(__file__).with_name("dist_worker.py")
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(worker), str(tmp_path / f"r{r}.json")],
                                      env=env))
    for p in procs:
        assert p.wait(timeout=300) == 0
    r0, r1 = (json.loads((tmp_path / f"r{r}.json").read_text()) for r in range(2))
    for k in ("digest", "nnz", "smem", "groups"):
        assert r0[k] == r1[k], k
    assert r0["nnz"] > 0 and r0["groups"] > 0


def _csr_apply(ip, ix, v, x):
    rows = np.repeat(np.arange(len(ip) - 1), np.diff(ip))
    out = np.zeros((len(ip) - 1,) + x.shape[1:])
    np.add.at(out, rows, v[:, None] * x[ix])
    return out


def test_domain_exchange_plan_reassembles_the_operator():
    """Host logic of the P_d > 1 exchange (parallel._DistSide): each rank
    multiplies its column block, then the send / recv / self maps route
    every partial to the owner of its output element.  Emulating the NCCL
    p2p with array copies, the owners' sums reproduce A x and A^T y."""
    from paper_2009_07226_b200 import geometry, pipeline
    g = geometry.make_geometry(40, 1, 24)
    og = O.make_geom(40, 1, 24)
    A = O.system_matrix(og)
    ip, ix, v = A.indptr, A.indices.astype(np.int32), A.values
    R, Cn = A.num_rows, A.num_cols
    P = 3
    tomo, sino = pipeline.hilbert_subdomains(g, 8, P)
    rng = np.random.default_rng(0)
    x = rng.random((Cn, 2))
    y = rng.random((R, 2))
    for direction in ("forward", "adjoint"):
        blocks, fps = [], []
        for r in range(P):
            if direction == "forward":
                bip, bix, bv, fp = pipeline.column_block(ip, ix, v, R, Cn, tomo[r].elements)
                blocks.append(_csr_apply(bip, bix, bv, x[tomo[r].elements]))
            else:
                bip, bix, bv, fp = pipeline.row_block_transposed(ip, ix, v, sino[r].elements)
                blocks.append(_csr_apply(bip, bix, bv, y[sino[r].elements]))
            fps.append(fp)
        owned = [s.elements for s in (sino if direction == "forward" else tomo)]
        ins = [s.elements for s in (tomo if direction == "forward" else sino)]
        sides = [parallel._DistSide(None, fps[r], owned[r], ins[r], fps, owned, r, "cpu")
                 for r in range(P)]
        full = (_csr_apply(ip, ix, v, x) if direction == "forward"
                else _csr_apply(*O_transpose(ip, ix, v, R, Cn), y))
        for q in range(P):
            me = sides[q]
            acc = np.zeros((len(owned[q]), 2))
            acc[me.self_dst.numpy()] += blocks[q][me.self_src.numpy()]
            for s in sorted(me.recv):
                sent = blocks[s][sides[s].send[q].numpy()]
                acc[me.recv[s].numpy()] += sent
            assert np.allclose(acc, full[owned[q]], rtol=1e-12, atol=1e-12), (direction, q)


def O_transpose(ip, ix, v, n_rows, n_cols):
    from paper_2009_07226_b200.pipeline import _transpose
    return _transpose(ip, ix, v, n_rows, n_cols)


def test_decompose_weighted_balances_siddon_work():
    """Equal-nnz cuts of the Hilbert tile curve (SURVEY §7 hard part 3):
    contiguous, complete, non-empty, and far better balanced than equal
    tile counts for the column (voxel) work of a parallel-beam operator."""
    import xct_oracle as O
    from paper_2009_07226_b200 import hilbert
    g = O.make_geom(64, 1, 64)
    A = O.system_matrix(g)
    w = np.bincount(A.indices, minlength=g.num_voxels).astype(np.float64)
    grid = hilbert.TileGrid("tomogram", 64, 64, 8)
    for P in (2, 4, 8):
        eq = hilbert.decompose(grid, P)
        wt = hilbert.decompose_weighted(grid, P, w)
        assert np.array_equal(np.sort(np.concatenate([s.elements for s in wt])),
                              np.arange(g.num_voxels))
        assert all(len(s.tiles) > 0 for s in wt)
        # contiguous along the curve: tiles in order, no gaps
        order = [tuple(c) for c in hilbert.pseudo_hilbert_cells(grid.tiles_x, grid.tiles_z)]
        assert [t for s in wt for t in s.tiles] == order
        imb = lambda parts: max(w[s.elements].sum() for s in parts) / (w.sum() / P)
        assert imb(wt) <= imb(eq) + 1e-9
        # within one tile of perfect balance
        tw = hilbert.tile_weights(grid, w)
        assert imb(wt) <= 1.0 + P * tw.max() / w.sum()
