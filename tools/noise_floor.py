#!/usr/bin/env python
"""Measure the reference algorithm's own CGLS order-noise floor at config 1
with the oracle (pinned bit-exact to the reference): per-row accumulation
orders drawn at random (any order is a valid staged-kernel order), 30
iterations, deviation from the reference's default run (golden c1 curve/x).
Writes tests/golden/noise_floor.json, read by the GPU parity tests to set
the native-order CGLS tolerances (2x the worst floor)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))
import xct_oracle as O  # noqa: E402
from conftest import load_golden  # noqa: E402


def main(seeds=5):
    gold = load_golden("c1")
    g = O.make_geom(180, 16, 128)
    A = O.system_matrix(g)
    y = O.measure(A, O.phantom("shepp-logan-like", 128, 16))
    orig = O.stage_order
    out = {}
    try:
        for prec in ("single", "mixed"):
            curve, xs = [], []
            for seed in range(1, seeds + 1):
                rng = np.random.default_rng(seed)

                def rnd_order(b, cap, parts, ff, p, rng=rng):
                    row = np.repeat(np.arange(b.num_rows), np.diff(b.indptr))
                    return row, np.lexsort((rng.random(len(b.indices)), row))
                O.stage_order = rnd_order
                r = O.cgls(O.Operator(A, g, prec, 16), y, 30, prec)
                curve.append(float(np.max(np.abs(np.array(r["residual"]) /
                                                 gold[f"cg_{prec}_residual"] - 1))))
                xs.append(float(np.linalg.norm(r["x"] - gold[f"cg_{prec}_x"]) /
                                np.linalg.norm(gold[f"cg_{prec}_x"])))
            out[prec] = {"curve_max_rel": curve, "x_rel_l2": xs}
            print(prec, out[prec])
    finally:
        O.stage_order = orig
    (ROOT / "tests" / "golden" / "noise_floor.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
