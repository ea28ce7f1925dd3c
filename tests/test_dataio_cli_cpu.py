"""Data formats and CLI surface on CPU: the XCT1 container,
PGM and CSV writers are byte-identical to the reference's own files
(tests/golden/dataio, written by tests/golden/make_golden_dataio.py with
the reference); error behaviour follows tests/test_cli.py of the reference."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2009_07226_b200 import dataio
from paper_2009_07226_b200.cli import main, slice_groups
from paper_2009_07226_b200.geometry import PHANTOM_KINDS, Volume, generate_phantom

import xct_oracle as O

GOLD = Path(__file__).resolve().parent / "golden" / "dataio"


@pytest.fixture()
def workdir(tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    return tmp_path


@pytest.mark.parametrize("tag", ["f8", "f4", "f2"])
@pytest.mark.parametrize("role", ["tomogram", "sinogram"])
def test_xct1_matches_reference_files(workdir, tag, role):
    data = np.load(GOLD / f"vol_{tag}_{role}.npy")
    ref = (GOLD / f"vol_{tag}_{role}.xct").read_bytes()
    dataio.write_volume("mine.xct", Volume(data, role=role))
    assert Path("mine.xct").read_bytes() == ref
    back = dataio.read_volume(GOLD / f"vol_{tag}_{role}.xct")
    assert back.role == role and back.data.dtype == data.dtype
    assert back.data.tobytes() == data.tobytes()
    part = dataio.read_slices(GOLD / f"vol_{tag}_{role}.xct", 1, 3)
    assert part.data.tobytes() == data[1:3].tobytes()


def test_pgm_csv_match_reference_files(workdir):
    dataio.write_pgm("img.pgm", np.load(GOLD / "pgm_src.npy"))
    assert Path("img.pgm").read_bytes() == (GOLD / "img.pgm").read_bytes()
    dataio.write_pgm("flat.pgm", np.full((2, 3), 0.5))
    assert Path("flat.pgm").read_bytes() == (GOLD / "flat.pgm").read_bytes()
    dataio.write_csv("t.csv", ["a", "b", "c"], [(1, 0.1, "x"), (2, 1e-20, "y")])
    assert Path("t.csv").read_bytes() == (GOLD / "table.csv").read_bytes()


@pytest.mark.parametrize("kind", PHANTOM_KINDS)
def test_cli_phantom_matches_reference_file(workdir, kind):
    assert main(["phantom", "--kind", kind, "--size", "16", "--slices", "2", "--seed", "3",
                 "--out", "p.xct"]) == 0
    assert Path("p.xct").read_bytes() == (GOLD / f"phantom_{kind}.xct").read_bytes()


def test_bad_files_rejected(workdir):
    Path("bad.xct").write_bytes(b"NOPE" + b"\x00" * 32)
    with pytest.raises(dataio.DatasetFormatError):
        dataio.read_volume("bad.xct")
    dataio.write_volume("t.xct", Volume(np.zeros((1, 4, 4)), role="tomogram"))
    Path("t.xct").write_bytes(Path("t.xct").read_bytes()[:-8])
    with pytest.raises(dataio.DatasetFormatError):
        dataio.read_volume("t.xct")
    raw = bytearray((GOLD / "vol_f4_tomogram.xct").read_bytes())
    raw[4] = 9                                     # unknown dtype code
    Path("c.xct").write_bytes(bytes(raw))
    with pytest.raises(dataio.DatasetFormatError):
        dataio.read_volume("c.xct")
    with pytest.raises(FileNotFoundError) as err:
        dataio.read_volume("absent.xct")
    assert "absent.xct" in str(err.value)
    with pytest.raises(dataio.DatasetFormatError):
        dataio.write_volume("i.xct", Volume(np.zeros((1, 2, 2), np.int32), role="tomogram"))


def test_manifest_roundtrip(workdir):
    Path("out.bin").write_bytes(b"abc")
    m = dataio.RunManifest(command="recon", arguments={"iters": 3}, seeds={"seed": 1})
    m.add_output("out.bin")
    m.save("m.json")
    back = dataio.RunManifest.load("m.json")
    assert back == m
    assert json.loads(Path("m.json").read_text())["outputs"]["out.bin"] == \
        "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"


def test_cli_errors_and_exit_codes(workdir, capsys):
    assert main(["phantom", "--kind", "uniform-disk", "--size", "8", "--frobnicate", "1",
                 "--out", "x.xct"]) != 0
    assert main(["transmogrify"]) != 0
    code = main(["export", "--in", "nope.xct", "--slice", "0", "--out", "o.pgm"])
    assert code == 2 and "nope.xct" in capsys.readouterr().err
    dataio.write_volume("z.xct", Volume(np.zeros((1, 6, 5)), role="tomogram"))
    assert main(["export", "--in", "z.xct", "--slice", "0", "--out", "z.pgm"]) == 0
    raw = Path("z.pgm").read_bytes()
    assert raw.startswith(b"P5\n5 6\n65535\n") and raw.endswith(b"\x00" * 60)
    assert main(["export", "--in", "z.xct", "--slice", "4", "--out", "z.pgm"]) == 2
    dataio.write_volume("t.xct", generate_phantom("uniform-disk", 16, 1))
    # role mismatch is a usage error before any device work
    assert main(["recon", "--in", "t.xct", "--geometry", "24,1,16", "--iters", "2",
                 "--out", "r.xct"]) == 2
    # no P_d fits a cap below the stage buffers (src/cli.py:108-110)
    assert main(["plan", "--geometry", "96,1,64", "--mem-cap", "1000", "--report", "p.csv"]) == 2


def test_slice_groups_rule():
    assert slice_groups(10, 3) == O.slice_groups(10, 3)
    assert slice_groups(3, 8) == [(0, 1), (1, 2), (2, 3)]


PLAN = Path(__file__).resolve().parent / "golden" / "plan"
PLAN_ARGS = {       # tests/golden/make_golden_plan.py, run with the reference CLI
    "whatif_c4": ["--geometry", "2048,1024,2048"],
    "whatif_nofit": ["--geometry", "96,1,64", "--pd", "30"],
    "whatif_cap": ["--geometry", "1024,256,1024", "--precision", "mixed",
                   "--mem-cap", "3000000000", "--ffactor", "8"],
}


@pytest.mark.parametrize("name", sorted(PLAN_ARGS))
def test_plan_whatif_matches_reference(workdir, capsys, name):
    """Analytic what-if path of `xct plan`: same P_d/P_b choice, memory model,
    stdout and CSV bytes as the reference CLI."""
    assert main(["plan", *PLAN_ARGS[name], "--report", f"{name}.csv"]) == 0
    assert Path(f"{name}.csv").read_bytes() == (PLAN / f"{name}.csv").read_bytes()
    assert capsys.readouterr().out == (PLAN / f"{name}.out").read_text()
