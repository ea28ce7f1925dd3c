"""Exchange byte accounting against the reference planner's
own outputs (tests/golden/comm_plans.npz, made by make_golden_comm.py from
src/comm.py:270-417 via src/pipeline.py:64-194).  Bytes, counts, element
lists and the transfer order are exact; level times are the same float sums
in the same order, so they are compared exactly too."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2009_07226_b200 import comm

GOLDEN = Path(__file__).resolve().parent / "golden" / "comm_plans.npz"


def _load():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["meta"]).decode())
    topos = {k: comm.Topology(**v) for k, v in meta["topologies"].items()}
    return z, meta["cases"], topos


Z, CASES, TOPOS = _load()
SIDE_NAMES = ("projection", "backprojection")


def _inputs(i, side, info):
    key = f"c{i}_{side}"
    fps = {p: Z[f"{key}_fp{p}"] for p in range(info["n_fp"])}
    own = {q: Z[f"{key}_own{q}"] for q in range(info["n_own"])}
    return key, fps, own


def check_report(got: comm.VolumeReport, want: dict):
    for f in ("ffactor", "element_bytes", "direct_bytes", "direct_inter_node_bytes",
              "hier_inter_node_bytes", "retained_bytes", "level_bytes", "level_times",
              "inter_node_reduction_pct"):
        assert getattr(got, f) == want[f], f
    assert [list(r) for r in got.level_rows()] == want["level_rows"]


@pytest.mark.parametrize("i", range(len(CASES)))
@pytest.mark.parametrize("side", SIDE_NAMES)
def test_planner_matches_reference(i, side):
    case = CASES[i]
    info = case["sides"][side]
    key, fps, own = _inputs(i, side, info)
    placement = comm.map_partitions(case["p_b"], case["p_d"], TOPOS[case["topology"]])
    planner = comm.plan_hierarchical if case["strategy"] == "hierarchical" else comm.plan_direct
    eb = {"double": 8, "single": 4, "half": 2, "mixed": 2}[case["precision"]]
    plan, report = planner(fps, own, placement, ffactor=case["ffactor"], elem_bytes=eb)
    check_report(report, info["report"])
    assert [lv.level for lv in plan.levels] == info["levels"]
    for lv in plan.levels:
        np.testing.assert_array_equal(lv.counts, Z[f"{key}_{lv.level}_counts"])
        pairs = Z[f"{key}_{lv.level}_pairs"]
        assert [tuple(p) for p in pairs.tolist()] == list(lv.transfers), lv.level
        for j, pr in enumerate(lv.transfers):
            np.testing.assert_array_equal(lv.transfers[pr], Z[f"{key}_{lv.level}_t{j}"])


def test_topology_parse_and_placement():
    t = comm.parse_topology("nodes=2 sockets=2 gpus=4 bw_socket=9e10 bw_node=4e10 "
                            "bw_inter=1e10 lat=3e-6")
    assert (t.num_nodes, t.gpus_per_node, t.total_gpus) == (2, 8, 16)
    pl = comm.map_partitions(2, 6, t)
    assert pl.slot(0) == (0, 0, 0) and pl.slot(5) == (0, 1, 1)
    assert pl.node_of(6) == 1 and pl.socket_of(11) == 3
    assert pl.group_pids(1) == list(range(6, 12))
    with pytest.raises(ValueError):
        comm.map_partitions(3, 8, t)
    with pytest.raises(ValueError):
        comm.parse_topology("nodes=2 bogus=1")
    with pytest.raises(ValueError):
        comm.Topology(bw_intra_socket=1e9, bw_intra_node=2e9)


def test_ownership_errors():
    pl = comm.map_partitions(1, 2, comm.default_topology())
    with pytest.raises(ValueError, match="duplicate"):
        comm.plan_direct({0: [0, 1]}, {0: [0, 1], 1: [1]}, pl)
    with pytest.raises(ValueError, match="no owner"):
        comm.plan_hierarchical({0: [0, 5]}, {0: [0, 1], 1: [2]}, pl)


def test_estimate_makespan():
    assert comm.estimate_makespan(1.0, 0.5, 2.0, 4, overlap=False) == 4 * 3.5
    assert comm.estimate_makespan(1.0, 0.5, 2.0, 4, overlap=True) == 3.5 + 3 * 2.0
    with pytest.raises(ValueError):
        comm.estimate_makespan(1.0, -1.0, 0.0, 1, overlap=True)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CASES)))
def test_assembled_volume_reports_match_reference(i):
    """`AssembledSystem.volume_reports()` of the B200 pipeline equals the
    reference's `{projection, backprojection}` reports (src/pipeline.py:192-194;
    tests/test_solver.py:265-273), and its footprints equal the reference's."""
    from paper_2009_07226_b200 import geometry, pipeline
    case = CASES[i]
    g = geometry.make_geometry(case["k"], case["n"], case["n"])
    cfg = pipeline.SystemConfig(precision=case["precision"], ffactor=case["ffactor"],
                                p_b=case["p_b"], p_d=case["p_d"],
                                topology=TOPOS[case["topology"]],
                                comm_strategy=case["strategy"],
                                stage_capacity_bytes=None, block_partitions=1)
    system = pipeline.assemble(g, cfg)
    reports = system.volume_reports()
    assert set(reports) == set(SIDE_NAMES)
    for side_name, side in (("projection", system.forward), ("backprojection", system.adjoint)):
        info = case["sides"][side_name]
        if case["p_d"] > 1:
            _, fps, _ = _inputs(i, side_name, info)
            for p, fp in enumerate(side.footprints):
                np.testing.assert_array_equal(np.asarray(fp), fps[p])
        check_report(reports[side_name], info["report"])


def _random_partition(rng, n_el, p_d):
    """Random ownership partition and overlapping footprints (some ranks
    empty, some elements held by many ranks)."""
    owner = rng.integers(0, p_d, n_el)
    own = {q: np.flatnonzero(owner == q) for q in range(p_d)}
    fps = {}
    for p in range(p_d):
        dens = rng.choice([0.0, 0.05, 0.3, 0.9])
        fps[p] = np.flatnonzero(rng.random(n_el) < dens)
    return fps, own


@pytest.mark.parametrize("seed", range(12))
def test_planner_matches_elementwise_oracle(seed):
    """Random topologies, P_b x P_d placements, ragged/empty footprints:
    the vectorized planner equals the element-by-element restatement of the
    reference (oracle.plan_levels) in every transfer list and its order."""
    import xct_oracle as O
    rng = np.random.default_rng(seed)
    topo = comm.Topology(num_nodes=int(rng.integers(2, 5)), sockets_per_node=int(rng.integers(1, 3)),
                         gpus_per_socket=int(rng.integers(1, 4)))
    p_d = int(rng.integers(1, topo.gpus_per_node * (topo.num_nodes // 2) + 1))
    p_b = max(1, topo.num_nodes // -(-p_d // topo.gpus_per_node))
    placement = comm.map_partitions(p_b, p_d, topo)
    assert list(placement.slots) == O.placement_slots(p_b, p_d, topo.num_nodes,
                                                      topo.sockets_per_node, topo.gpus_per_socket)
    fps, own = _random_partition(rng, int(rng.integers(1, 400)), p_d)
    for hier in (False, True):
        planner = comm.plan_hierarchical if hier else comm.plan_direct
        plan, rep = planner(fps, own, placement, ffactor=3, elem_bytes=2)
        want, retained = O.plan_levels({p: f.tolist() for p, f in fps.items()},
                                       {q: o.tolist() for q, o in own.items()},
                                       placement.slots, topo.sockets_per_node, hier)
        for lv, (name, t) in zip(plan.levels, want):
            assert lv.level == name
            got = {k: v.tolist() for k, v in lv.transfers.items() if k[0] != k[1]}
            assert list(got) == list(t) and got == t, name
            assert lv.volume_elements() == sum(len(v) for v in t.values())
        assert [b // 6 for b in rep.retained_bytes] == retained


@pytest.mark.parametrize("i", range(len(CASES)))
def test_oracle_planner_pinned_to_reference(i):
    """The element-by-element oracle itself reproduces the reference's
    golden transfer lists (pins the oracle, tests/golden/comm_plans.npz)."""
    import xct_oracle as O
    case = CASES[i]
    topo = TOPOS[case["topology"]]
    pl = comm.map_partitions(case["p_b"], case["p_d"], topo)
    for side in SIDE_NAMES:
        info = case["sides"][side]
        key, fps, own = _inputs(i, side, info)
        want, _ = O.plan_levels({p: f.tolist() for p, f in fps.items()},
                                {q: o.tolist() for q, o in own.items()},
                                list(pl.slots), topo.sockets_per_node,
                                case["strategy"] == "hierarchical")
        for name, t in want:
            pairs = [tuple(p) for p in Z[f"{key}_{name}_pairs"].tolist()]
            ref = {pr: Z[f"{key}_{name}_t{j}"].tolist() for j, pr in enumerate(pairs)
                   if pr[0] != pr[1]}
            assert list(ref) == list(t) and ref == t, (side, name)
