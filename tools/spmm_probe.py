#!/usr/bin/env python
"""Time (and, under ncu, profile) the staged SpMM alone: assemble a config,
then run `reps` forward and `reps` back projections on device-resident
chunked inputs and print per-launch CUDA-event times and achieved GB/s.

  python tools/spmm_probe.py --config c2 --reps 3 [--warps 16] [--smem 98304]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--warps", type=int, default=16)
    ap.add_argument("--smem", type=int, default=96 * 1024)
    ap.add_argument("--slices", type=int, default=None)
    ap.add_argument("--order", default="native")
    ap.add_argument("--ppl", type=int, default=None)
    ap.add_argument("--groups", default="16", help="chunk_group values to sweep")
    ap.add_argument("--row-group", type=int, default=None)
    ap.add_argument("--ffactor", type=int, default=16)
    ap.add_argument("--contract", default="auto", help="auto | 0 | 1 | sweep")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.precision:
        cfg["precision"] = args.precision
    S = args.slices or cfg["slices"]
    import torch
    from paper_2009_07226_b200 import engine, geometry, matrixstore, pipeline
    dev = torch.device("cuda", 0)
    g = geometry.make_geometry(cfg["k"], S, cfg["n"])
    t0 = time.perf_counter()
    system = pipeline.assemble(g, pipeline.SystemConfig(
        precision=cfg["precision"], ffactor=args.ffactor, order=args.order, warps_per_cta=args.warps,
        smem_budget=args.smem, pieces_per_lane=args.ppl, row_group=args.row_group))
    t_asm = time.perf_counter() - t0
    nnz = system.matrix.nnz
    geometry.clear_matrix_cache()
    torch.cuda.empty_cache()
    prec = cfg["precision"]
    sd = {"double": torch.float64, "single": torch.float32}.get(prec, torch.float16)
    od = torch.float64 if prec == "double" else torch.float32
    eb = matrixstore.element_bytes(prec)
    out = {"config": args.config, "precision": prec, "slices": S, "nnz": nnz,
           "row_group": args.row_group,
           "assemble_s": t_asm, "warps": args.warps, "smem": args.smem, "ppl": args.ppl}
    for name, side in (("forward", system.forward), ("adjoint", system.adjoint)):
        blk = side.blocks[0]
        n_chunks = -(-S // args.ffactor)
        x = torch.rand((n_chunks, blk.n_in, blk.f_dev), device=dev, dtype=sd) * 0.5
        y = torch.empty((n_chunks, blk.n_out, blk.f_dev), dtype=od, device=dev)
        fac = torch.ones(n_chunks, dtype=torch.float64, device=dev)
        contracts = {"auto": [blk.contract], "0": [False], "1": [True],
                     "sweep": [False, True]}[args.contract]
        if prec != "single":
            contracts = [False]
        sweep = {}
        ref_y = None
        for cc in contracts:
            for G in [int(v) for v in args.groups.split(",")]:
                matrixstore.set_execution(blk, cc, G)
                times = []
                for _ in range(args.reps):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    engine.apply_side(blk, x, y, row_stride=blk.f_dev,
                                      chunk_stride=blk.n_out * blk.f_dev,
                                      valid_cols=n_chunks * blk.f_dev, ffactor_out=blk.f_dev,
                                      factors=fac)
                    e1.record()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1) / 1e3)
                if ref_y is None:
                    ref_y = y.clone()
                    dev_rel = 0.0
                else:
                    dev_rel = float((y - ref_y).norm() / ref_y.norm())
                sweep[f"contract={int(cc)},G={G}"] = {"ms": round(min(times) * 1e3, 3),
                                                      "rel_vs_first": dev_rel}
        t = min(times)
        bytes_alg = blk.nnz * (2 + eb) * n_chunks + (blk.n_in + blk.n_out) * S * eb
        out[name] = {"sweep": sweep, "ms": [round(v * 1e3, 3) for v in times],
                     "gflops": 2 * blk.nnz * S / t / 1e9,
                     "alg_gbs": bytes_alg / t / 1e9, "bytes_alg": bytes_alg,
                     "padded_ratio": blk.padded_entries / blk.nnz,
                     "slots_per_nnz": int(blk.info.n_slots) / blk.nnz,
                     "n_cta": int(blk.info.n_cta), "n_groups": int(blk.info.n_groups),
                     "rows_per_cta": int(blk.info.rows_per_cta),
                     "smem_bytes": blk.smem_bytes}
        del x, y, ref_y
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
