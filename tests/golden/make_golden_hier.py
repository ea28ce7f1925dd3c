"""Reference outputs of the P_d > 1 operator with the reference's DEFAULT
exchange, comm_strategy="hierarchical" (socket -> node -> global levels over
the default 4 x 2 x 3 topology, src/comm.py:344-472), which sums partials in
another order than the direct plan.  Run in the build container:

    python tests/golden/make_golden_hier.py    -> tests/golden/pipeline_g64_hier.npz
"""
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from xct import geometry, pipeline  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    g64 = geometry.make_geometry(96, 1, 64)
    gold = np.load(OUT / "pipeline_g64.npz")
    x64, y64 = gold["x64"].astype(np.float32), gold["y64"]
    out = {}
    for prec in ("double", "single", "mixed"):
        for p_d in (4, 6):
            sysm = pipeline.assemble(g64, pipeline.SystemConfig(
                precision=prec, ffactor=4, p_d=p_d, comm_strategy="hierarchical"))
            out[f"g64_pd{p_d}_fwd_{prec}"] = sysm.apply_forward(x64)[0]
            out[f"g64_pd{p_d}_adj_{prec}"] = sysm.apply_adjoint(y64)[0]
            d = pipeline.assemble(g64, pipeline.SystemConfig(
                precision=prec, ffactor=4, p_d=p_d, comm_strategy="direct"))
            diff = int(np.sum(d.apply_forward(x64)[0] != out[f"g64_pd{p_d}_fwd_{prec}"]))
            print(prec, p_d, "forward elements differing from the direct plan:", diff)
    np.savez_compressed(OUT / "pipeline_g64_hier.npz", **out)


if __name__ == "__main__":
    main()
