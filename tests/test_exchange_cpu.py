"""The native domain partition's exchange host logic (domain.py) on CPU:
gloo, world sizes 2 and 3, real p2p messages.  Forward: every owned ray
sums its partials owner-first, then senders ascending -- exactly the
reference's direct-plan order (src/comm.py:420-472) -- and A x is
reassembled; adjoint: the gathered inputs equal y on the footprint and A^T y
is reassembled without any partial-tomogram reduction."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import xct_oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_native_exchange_gloo(tmp_path, world):
    port = _free_port()
    worker = Path(__file__).with_name("dist_exchange_worker.py")
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(worker), str(tmp_path / f"r{r}.npz")],
                                      env=env))
    for p in procs:
        assert p.wait(timeout=300) == 0
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    k, n, F = 40, 24, 3
    g = O.make_geom(k, 1, n)
    A = O.system_matrix(g)
    rng = np.random.default_rng(7)
    x = rng.random((g.num_voxels, F)).astype(np.float32)
    y = rng.random((g.num_rays, F)).astype(np.float32)
    dense = A.dense()
    # forward: owners' sums == the direct-plan reduction of the partials
    owner_of = {}
    for r in res:
        for i, e in enumerate(r["own_rows"]):
            owner_of[int(e)] = (int(r["rank"]), i)
    want = np.zeros((g.num_rays, F), np.float32)
    for e, (q, i) in owner_of.items():
        acc = None
        for s in [q] + [s for s in range(world) if s != q]:
            fp = res[s]["fp"]
            hit = np.nonzero(fp == e)[0]
            if len(hit):
                v = res[s]["part"][hit[0]]
                acc = v.copy() if acc is None else acc + v
        if acc is not None:
            want[e] = acc
    got = np.zeros_like(want)
    for r in res:
        got[r["own_rows"]] = r["o"]
    assert np.array_equal(got, want)
    assert np.allclose(got, dense @ x.astype(np.float64), rtol=1e-5, atol=1e-4)
    # adjoint: the owned voxels are complete
    xt = np.zeros((g.num_voxels, F))
    for r in res:
        xt[r["cols"]] = r["xo"]
    assert np.allclose(xt, dense.T @ y.astype(np.float64), rtol=1e-10, atol=1e-10)
