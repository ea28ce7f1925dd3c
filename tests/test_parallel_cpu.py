"""Multi-process host logic on CPU (gloo, world_size 2): the slice-batch
rule and the broadcast of a staged operator side from the building rank."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

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
