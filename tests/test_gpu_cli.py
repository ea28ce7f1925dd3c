"""The xct CLI on the B200 backend, mirroring the
reference's tests/test_cli.py, plus parity with files the reference CLI
wrote (tests/golden/dataio/cli_*, tests/golden/make_golden_dataio.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2009_07226_b200 import dataio
from paper_2009_07226_b200.cli import main

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "dataio"


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture()
def workdir(tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    return tmp_path


def test_project_and_recon_match_reference_cli(workdir):
    """Same files in, same commands: the sinogram (float64, noise from the
    same seeded PCG64 stream) and the reconstructions of the reference CLI
    (P_d = 4, 6 CGLS iterations; --order reference)."""
    assert main(["project", "--geometry", "24,2,16", "--in", str(GOLD / "cli_ph.xct"),
                 "--noise", "0.01", "--seed", "4", "--out", "s.xct"]) == 0
    mine, ref = dataio.read_volume("s.xct"), dataio.read_volume(GOLD / "cli_sino.xct")
    assert mine.role == ref.role == "sinogram" and mine.data.shape == ref.data.shape
    assert rel(mine.data, ref.data) <= 1e-14
    tol = {"double": 1e-9, "single": 1e-5, "mixed": 2e-3}
    for prec in ("double", "single", "mixed"):
        assert main(["recon", "--in", str(GOLD / "cli_sino.xct"), "--geometry", "24,2,16",
                     "--iters", "6", "--pd", "4", "--precision", prec, "--seed", "3",
                     "--order", "reference", "--out", f"r_{prec}.xct",
                     "--residuals", f"res_{prec}.csv"]) == 0
        r = dataio.read_volume(f"r_{prec}.xct")
        g = dataio.read_volume(GOLD / f"cli_rec_{prec}.xct")
        assert r.data.dtype == g.data.dtype and r.data.shape == g.data.shape
        assert rel(r.data, g.data) <= tol[prec], (prec, rel(r.data, g.data))
        cur = [l.split(",") for l in Path(f"res_{prec}.csv").read_text().splitlines()]
        gold = [l.split(",") for l in (GOLD / f"cli_res_{prec}.csv").read_text().splitlines()]
        assert cur[0] == gold[0] and len(cur) == len(gold)
        for a, b in zip(cur[1:], gold[1:]):
            assert abs(float(a[2]) / float(b[2]) - 1) <= 10 * tol[prec], (prec, a, b)


def test_phantom_project_recon_export(workdir):
    assert main(["phantom", "--kind", "uniform-disk", "--size", "32", "--slices", "2",
                 "--out", "ph.xct"]) == 0
    assert main(["project", "--geometry", "48,2,32", "--in", "ph.xct", "--noise", "0",
                 "--out", "sino.xct"]) == 0
    assert main(["recon", "--in", "sino.xct", "--geometry", "48,2,32", "--iters", "12",
                 "--precision", "double", "--ffactor", "2", "--pd", "4", "--out", "rec.xct",
                 "--manifest", "man.json", "--residuals", "res.csv"]) == 0
    assert main(["export", "--in", "rec.xct", "--slice", "0", "--out", "rec.pgm"]) == 0
    rec, ph = dataio.read_volume("rec.xct"), dataio.read_volume("ph.xct")
    # the reference's own test asserts < 0.1, but the reference itself gives
    # 0.2280 on this run (its one failing test: 211/212 pass);
    # we reproduce the reference's value
    assert abs(np.abs(rec.data - ph.data).max() - 0.2280) < 0.01
    lines = Path("res.csv").read_text().splitlines()
    assert lines[0] == "iteration,double_seconds,double_rel_residual" and len(lines) == 13
    man = json.loads(Path("man.json").read_text())
    assert man["counters"]["projections"] == 12 and man["counters"]["backprojections"] == 13
    assert Path("rec.pgm").read_bytes().startswith(b"P5\n32 32\n65535\n")


def test_end_to_end_residual_drops_and_wrong_geometry(workdir):
    assert main(["phantom", "--kind", "shepp-logan-like", "--size", "32", "--out", "ph.xct"]) == 0
    assert main(["project", "--geometry", "48,1,32", "--in", "ph.xct", "--out", "s.xct"]) == 0
    for prec in ("double", "single", "mixed"):
        assert main(["recon", "--in", "s.xct", "--geometry", "48,1,32", "--iters", "30",
                     "--precision", prec, "--out", "r.xct", "--residuals", "res.csv"]) == 0
        last = Path("res.csv").read_text().splitlines()[-1]
        assert float(last.split(",")[2]) < 1e-2, prec
    assert main(["project", "--geometry", "24,1,16", "--in", "ph.xct", "--out", "x.xct"]) == 2
    assert main(["recon", "--in", "s.xct", "--geometry", "40,1,32", "--out", "x.xct"]) == 2


def test_determinism_workers_rerun_and_manifest_replay(workdir):
    assert main(["phantom", "--kind", "random-blobs", "--size", "16", "--slices", "2",
                 "--seed", "9", "--out", "ph.xct"]) == 0
    assert main(["project", "--geometry", "24,2,16", "--in", "ph.xct", "--noise", "0.01",
                 "--seed", "4", "--out", "sino.xct"]) == 0
    for out, workers in (("a.xct", 1), ("b.xct", 4), ("c.xct", 1)):
        assert main(["recon", "--in", "sino.xct", "--geometry", "24,2,16", "--iters", "6",
                     "--pd", "4", "--workers", str(workers), "--seed", "3",
                     "--precision", "mixed", "--out", out, "--manifest", out + ".json"]) == 0
    a, b, c = (Path(p).read_bytes() for p in ("a.xct", "b.xct", "c.xct"))
    assert a == b == c
    for extra in ([], ["--pb", "2"]):
        assert main(["recon", "--in", "sino.xct", "--geometry", "24,2,16", "--iters", "4",
                     "--out", "r1.xct", "--manifest", "m1.json"] + extra) == 0
        args = dataio.RunManifest.load("m1.json").arguments
        replay = ["recon", "--in", args["in"], "--geometry", args["geometry"],
                  "--iters", str(args["iters"]), "--pb", str(args["pb"]),
                  "--out", "r2.xct", "--manifest", "m2.json"]
        assert main(replay) == 0
        assert Path("r1.xct").read_bytes() == Path("r2.xct").read_bytes()
        assert dataio.RunManifest.load("m1.json").outputs["r1.xct"] == \
            dataio.RunManifest.load("m2.json").outputs["r2.xct"]


def test_bench_sweep(workdir):
    assert main(["bench", "--geometry", "24,1,32", "--ffactor-sweep", "1..8",
                 "--report", "bench.csv"]) == 0
    lines = Path("bench.csv").read_text().splitlines()
    assert lines[0] == "ffactor,nnz,flops,bytes,intensity" and len(lines) == 9
    ai = [float(l.split(",")[4]) for l in lines[1:]]
    assert all(b > a for a, b in zip(ai, ai[1:]))
    assert int(lines[1].split(",")[2]) == 2 * int(lines[1].split(",")[1])


PLAN = Path(__file__).resolve().parent / "golden" / "plan"


@pytest.mark.parametrize("name,args", [
    ("desk_pd6", ["--geometry", "96,1,64", "--pd", "6", "--precision", "mixed",
                  "--ffactor", "4"]),
    ("desk_auto_topo", ["--geometry", "60,3,40", "--mem-cap", "150000", "--stage-capacity",
                        "16384", "--block-partitions", "2", "--topology", "TOPO",
                        "--precision", "single"]),
])
def test_plan_desk_report_matches_reference(workdir, capsys, name, args):
    """Desk path of `xct plan`: the per-level communication report of the
    operator assembled on the GPU equals the reference CLI's CSV and stdout
    byte for byte (tests/golden/make_golden_plan.py)."""
    args = [str(PLAN / "topo.txt") if a == "TOPO" else a for a in args]
    assert main(["plan", *args, "--report", f"{name}.csv"]) == 0
    assert Path(f"{name}.csv").read_bytes() == (PLAN / f"{name}.csv").read_bytes()
    assert capsys.readouterr().out == (PLAN / f"{name}.out").read_text()
