"""Golden files of the data formats (XCT1 container, PGM, CSV, manifest
fields) written by the REFERENCE's own xct.dataio (src/dataio.py) and the
reference CLI's phantom command.  Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_dataio.py

Writes tests/golden/dataio/*.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from xct import dataio, geometry  # noqa: E402
from xct.cli import main  # noqa: E402

OUT = Path(__file__).resolve().parent / "dataio"


def run():
    OUT.mkdir(exist_ok=True)
    rng = np.random.default_rng(7)
    for dt, tag in ((np.float64, "f8"), (np.float32, "f4"), (np.float16, "f2")):
        for role in ("tomogram", "sinogram"):
            data = (rng.random((3, 5, 4)) * 4 - 2).astype(dt)
            dataio.write_volume(OUT / f"vol_{tag}_{role}.xct", geometry.Volume(data, role=role))
            np.save(OUT / f"vol_{tag}_{role}.npy", data)
    img = rng.random((6, 7)) * 3 - 1
    np.save(OUT / "pgm_src.npy", img)
    dataio.write_pgm(OUT / "img.pgm", img)
    dataio.write_pgm(OUT / "flat.pgm", np.full((2, 3), 0.5))
    dataio.write_csv(OUT / "table.csv", ["a", "b", "c"], [(1, 0.1, "x"), (2, 1e-20, "y")])
    # a tiny end-to-end run of the reference CLI: phantom -> project -> recon
    ph, sino, rec = (str(OUT / n) for n in ("cli_ph.xct", "cli_sino.xct", "cli_rec.xct"))
    assert main(["phantom", "--kind", "random-blobs", "--size", "16", "--slices", "2",
                 "--seed", "9", "--out", ph]) == 0
    assert main(["project", "--geometry", "24,2,16", "--in", ph, "--noise", "0.01",
                 "--seed", "4", "--out", sino]) == 0
    for prec in ("double", "single", "mixed"):
        assert main(["recon", "--in", sino, "--geometry", "24,2,16", "--iters", "6",
                     "--pd", "4", "--precision", prec, "--seed", "3",
                     "--out", str(OUT / f"cli_rec_{prec}.xct"),
                     "--residuals", str(OUT / f"cli_res_{prec}.csv")]) == 0
    for kind in geometry.PHANTOM_KINDS:
        assert main(["phantom", "--kind", kind, "--size", "16", "--slices", "2",
                     "--seed", "3", "--out", str(OUT / f"phantom_{kind}.xct")]) == 0


if __name__ == "__main__":
    run()
