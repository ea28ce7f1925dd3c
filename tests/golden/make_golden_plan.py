"""Golden outputs of the REFERENCE `xct plan` (src/cli.py:101-156).

Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_plan.py

Writes ``tests/golden/plan/<case>.csv`` and ``<case>.out`` (stdout) plus the
topology file the cases use.  Cases named ``desk_*`` assemble the operator
(GPU on the B200 side); ``whatif_*`` are the analytic path.
"""

from __future__ import annotations

import contextlib
import io
import os
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from xct.cli import main  # noqa: E402

OUT = Path(__file__).resolve().parent / "plan"
TOPO = "nodes=4 sockets=2 gpus=2 bw_socket=90e9 bw_node=40e9 bw_inter=10e9 lat=2e-6\n"

CASES = {
    "whatif_c4": ["--geometry", "2048,1024,2048"],
    "whatif_nofit": ["--geometry", "96,1,64", "--pd", "30"],
    "whatif_cap": ["--geometry", "1024,256,1024", "--precision", "mixed",
                   "--mem-cap", "3000000000", "--ffactor", "8"],
    "desk_pd6": ["--geometry", "96,1,64", "--pd", "6", "--precision", "mixed", "--ffactor", "4"],
    "desk_auto_topo": ["--geometry", "60,3,40", "--mem-cap", "150000", "--stage-capacity", "16384", "--block-partitions", "2",
                       "--topology", "TOPO", "--precision", "single"],
}


def main_():
    OUT.mkdir(exist_ok=True)
    (OUT / "topo.txt").write_text(TOPO, encoding="ascii")
    os.chdir(OUT)
    for name, argv in CASES.items():
        argv = ["plan", *[("topo.txt" if a == "TOPO" else a) for a in argv],
                "--report", f"{name}.csv"]
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = main(argv)
        assert rc == 0, (name, rc)
        (OUT / f"{name}.out").write_text(buf.getvalue(), encoding="ascii")
        print(name, buf.getvalue().strip().splitlines()[0])


if __name__ == "__main__":
    main_()
