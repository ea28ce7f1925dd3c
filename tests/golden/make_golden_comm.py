"""Golden vectors for the exchange byte accounting, made by
running the REFERENCE planner (src/comm.py:270-417) and pipeline
(src/pipeline.py:64-194).

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_comm.py

Writes ``tests/golden/comm_plans.npz``: the inputs (footprints, ownership,
topology) and the reference's VolumeReport fields, per-level count matrices
and transfer lists (pair order = the reference's dict order).
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from xct import comm, geometry, pipeline  # noqa: E402

OUT = Path(__file__).resolve().parent / "comm_plans.npz"

TOPOLOGIES = {
    "default": comm.default_topology(),
    "dense": comm.parse_topology("nodes=4 sockets=2 gpus=2 bw_socket=90e9 bw_node=40e9 "
                                 "bw_inter=10e9 lat=2e-6 stage_overhead=1.5"),
    "flat": comm.parse_topology("nodes=8 sockets=1 gpus=1 bw_socket=25e9 bw_node=25e9 "
                                "bw_inter=25e9 lat=5e-6"),
}

# (geometry k, n, p_b, p_d, precision, ffactor, topology, strategy)
CASES = [
    (48, 32, 1, 6, "mixed", 4, "default", "hierarchical"),
    (48, 32, 1, 6, "single", 16, "default", "direct"),
    (90, 64, 1, 12, "single", 16, "default", "hierarchical"),
    (60, 40, 2, 5, "double", 8, "dense", "hierarchical"),
    (36, 24, 1, 7, "half", 3, "flat", "hierarchical"),
    (40, 32, 1, 1, "single", 16, "default", "hierarchical"),
]


def main():
    blob, meta = {}, []
    for i, (k, n, p_b, p_d, prec, ff, topo_name, strat) in enumerate(CASES):
        g = geometry.make_geometry(k, n, n)
        cfg = pipeline.SystemConfig(precision=prec, ffactor=ff, p_b=p_b, p_d=p_d,
                                    topology=TOPOLOGIES[topo_name], comm_strategy=strat,
                                    stage_capacity_bytes=None, block_partitions=1)
        system = pipeline.assemble(g, cfg)
        case = dict(k=k, n=n, p_b=p_b, p_d=p_d, precision=prec, ffactor=ff,
                    topology=topo_name, strategy=strat, sides={})
        for side_name, side in (("projection", system.forward), ("backprojection", system.adjoint)):
            key = f"c{i}_{side_name}"
            for p, fp in side.footprints.items():
                blob[f"{key}_fp{p}"] = np.asarray(fp, np.int64)
            for q, own in side.ownership.items():
                blob[f"{key}_own{q}"] = np.asarray(own, np.int64)
            r = side.report
            levels = []
            for lv in side.plan.levels:
                blob[f"{key}_{lv.level}_counts"] = lv.counts
                pairs = list(lv.transfers)
                blob[f"{key}_{lv.level}_pairs"] = np.array(pairs, np.int64).reshape(-1, 2)
                for j, pr in enumerate(pairs):
                    blob[f"{key}_{lv.level}_t{j}"] = np.asarray(lv.transfers[pr], np.int64)
                levels.append(lv.level)
            case["sides"][side_name] = dict(
                levels=levels, n_fp=len(side.footprints), n_own=len(side.ownership),
                report=dict(ffactor=r.ffactor, element_bytes=r.element_bytes,
                            direct_bytes=r.direct_bytes,
                            direct_inter_node_bytes=r.direct_inter_node_bytes,
                            level_bytes=r.level_bytes, level_times=r.level_times,
                            hier_inter_node_bytes=r.hier_inter_node_bytes,
                            retained_bytes=r.retained_bytes,
                            inter_node_reduction_pct=r.inter_node_reduction_pct,
                            level_rows=[list(x) for x in r.level_rows()]))
        meta.append(case)
    topo = {k: dict(vars(t)) for k, t in TOPOLOGIES.items()}
    blob["meta"] = np.frombuffer(json.dumps({"cases": meta, "topologies": topo}).encode(),
                                 np.uint8)
    np.savez_compressed(OUT, **blob)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(CASES)} cases)")


if __name__ == "__main__":
    main()
