#!/usr/bin/env python
"""Benchmark of the B200 XCT hot path: CGLS iterations (1 projection + 1
back projection + vector updates) on the staged sm_100a SpMM.

Metric (BASELINE.json): SpMM GFLOPS & CG s/iter.  A step is one CGLS
iteration over the whole slice batch; value = 2 applications x 2*nnz*S
flops / device seconds per iteration (whole job, all ranks).  Extra keys:
cg_s_per_iter, voxels_per_s, kernel-only SpMM GFLOPS, the roofline of the
SpMM kernel against measured HBM bandwidth, the CPU baseline (the oracle
port on an angle subset of the same geometry, extrapolated) and an
end-to-end number through the public API (cgls_solve on host arrays).

Multi-GPU (torchrun): slice-batch partitioning P_b = N (src/cli.py:158-200):
each rank reconstructs its own slice group of the same geometry, no
data-path collective; timing is max over ranks ("scaling": "weak").

  python bench.py [--config c2] [--steps K] [--warmup W] [--impl b200|reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # BASELINE.json configs; c2 is the single-GPU roofline workload
    "c1": dict(n=128, k=180, slices=16, precision="single", iters=30,
               desc="128x128 Shepp-Logan, 180 angles, 16 slices, FP32 CG"),
    "c2": dict(n=1024, k=1024, slices=256, precision="single", iters=50,
               desc="1024x1024, 1024 angles, 256 slices per GPU, FP32 CG"),
    "c2m": dict(n=1024, k=1024, slices=256, precision="mixed", iters=50,
                desc="1024x1024, 1024 angles, 256 slices per GPU, FP16 storage"),
    "c5": dict(n=2048, k=2048, slices=1024, precision="mixed", iters=30, strong=True,
               desc="2048x2048, 2048 angles, 1024 slices total, FP16 storage"),
    "c4": dict(n=2048, k=2048, slices=1024, precision="single", iters=30, strong=True,
               desc="2048x2048, 2048 angles, 1024 slices total, FP32 (domain-partitioned)"),
    "c3": dict(n=1024, k=1024, slices=2048, precision="single", iters=50, strong=True,
               desc="1024x1024, 1024 angles, 2048 slices total, slice batch, FP32"),
}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return False
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)
        return False

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit()
                else None, "reasons": reasons, "samples": len(self.rows)}


def make_problem(cfg, slices):
    """Shepp-Logan phantom (identical slices, src/geometry.py:337-339) and
    y = A x in float64 on the device (Siddon streamed over view chunks).
    Returns the one distinct sinogram column; the (rays, slices) problem is
    a zero-stride host view of it."""
    from paper_2009_07226_b200 import geometry
    g = geometry.make_geometry(cfg["k"], slices, cfg["n"])
    ph = geometry.generate_phantom("shepp-logan-like", cfg["n"], 1).slices_as_columns()
    return g, geometry.project_f64(g, ph.astype(np.float64))     # (rays, 1)


def cpu_baseline(cfg, slices, sample_angles=16, sample_slices=16):
    """The oracle port timed on an angle subset of the same geometry
    (BASELINE.md §3): K' views and S' slices, one forward + one back
    projection + the CG vector updates, extrapolated by (K/K')(S/S')."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import xct_oracle as O
    K, N = cfg["k"], cfg["n"]
    kp, sp = min(sample_angles, K), min(sample_slices, slices)
    g = O.make_geom(kp, sp, N, 0.0, kp * math.pi / K)
    t0 = time.perf_counter()
    A = O.system_matrix(g)
    t_build = time.perf_counter() - t0
    op = O.Operator(A, g, cfg["precision"], 16)
    rng = np.random.default_rng(0)
    x = rng.random((A.num_cols, sp)).astype(np.float32)
    yv = rng.random((A.num_rows, sp)).astype(np.float32)
    op.forward(x)
    op.adjoint(yv)                         # table construction (= assembly) untimed
    t0 = time.perf_counter()
    q, _ = op.forward(x)
    s, _ = op.adjoint(yv)
    a = np.float32(0.5)
    _ = x + a * x
    _ = yv - a * yv
    _ = x + a * x
    t_iter = time.perf_counter() - t0
    scale = (K / kp) * (slices / sp)
    return dict(t_iter_sample=t_iter, t_iter_extrap=t_iter * scale, nnz_sample=A.nnz,
                t_build_sample=t_build, kp=kp, sp=sp, scale=scale)


def _reference_worker(job):
    """One host core's share of the reference arm: the oracle port's CGLS
    iteration on the angle/slice sample, warmup + steps times."""
    cfg, total, n = job
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    return [cpu_baseline(cfg, total) for _ in range(n)]


def run_reference_arm(args, cfg, ws, rank):
    """--impl reference: the reference CPU path (the oracle port of
    src/engine.py + src/solver.py) on all host cores.  The reference runs
    one process per slice group (P_b, src/cli.py:158-200) and each group is
    independent, so every core times the same bounded sample (an exact
    angle subset) and the cores' rates add up."""
    if rank != 0:
        return
    import multiprocessing as mp
    total = cfg["slices"] if cfg.get("strong") else cfg["slices"] * ws
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    n = args.warmup + args.steps
    with mp.get_context("fork").Pool(cores) as pool:
        runs = pool.map(_reference_worker, [(cfg, total, n)] * cores)
    r = runs[0][-1]
    nnz_full = int(round(r["nnz_sample"] * cfg["k"] / r["kp"]))
    # per core: median extrapolated time of one full-workload iteration;
    # all cores together finish one iteration in 1 / sum(1 / t_core)
    t_core = [statistics.median([x["t_iter_extrap"] for x in run[args.warmup:]]) for run in runs]
    t = 1.0 / sum(1.0 / x for x in t_core)
    gflops = 4.0 * nnz_full * total / t / 1e9
    line = {"impl": "reference", "metric": metric_name(cfg), "value": gflops, "unit": "GFLOPS",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg.get("strong") else "weak",
            "vs_baseline": None, "dtype": "f32" if cfg["precision"] == "single" else "f16/f32",
            "data": "synthetic", "config": config_block(cfg, ws),
            "cg_s_per_iter": t,
            "cpu_baseline": {"value": gflops, "unit": "GFLOPS", "cores": cores, "kind": "port",
                             "sample": f"oracle port on {cores} host cores (one slice group "
                                       f"per core), each: views 0..{r['kp'] - 1} of {cfg['k']} "
                                       f"(bit-exact angle subset), {r['sp']} slices, one CGLS "
                                       f"iteration, extrapolated x{r['scale']:.0f}",
                             "per_core_s_per_iter": t_core},
            "e2e": {"value": gflops, "unit": "GFLOPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _global_nnz(system):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(system.forward.block.nnz)], dtype=torch.float64,
                     device=system.device)
    dist.all_reduce(t)
    return t.item()


def metric_name(cfg):
    per = "slices" if cfg.get("strong") else "slices/GPU"
    return (f"SpMM GFLOPS & CG s/iter ({cfg['n']}^2 x {cfg['slices']} {per}, "
            f"{cfg['k']} angles, {cfg['precision']})")


def config_block(cfg, ws):
    total = cfg["slices"] if cfg.get("strong") else cfg["slices"] * ws
    return {"workload": cfg["desc"], "n": cfg["n"], "angles": cfg["k"],
            # domain partition: every GPU holds all slices of its image/sinogram tiles
            "slices_per_gpu": (cfg["slices"] if not cfg.get("strong") or cfg.get("domain")
                               else -(-total // ws)),
            "total_slices": total,
            "precision": cfg["precision"], "ffactor": 16, "step": "one CGLS iteration",
            "parallelism": (f"image-domain P_d={ws}" if cfg.get("domain") else
                            f"slice-batch P_b={ws}"), "l2": "inputs >> L2 (matrix "
            "streamed from HBM every application), no flush needed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default=None)
    ap.add_argument("--order", default="native")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-iters", type=int, default=None)
    ap.add_argument("--partition", default="slices", choices=["slices", "domain"],
                    help="multi-GPU: slice batch (P_b, default) or image-domain tiles "
                         "with the NCCL partial-result exchange (P_d)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.precision:
        cfg["precision"] = args.precision
    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, cfg, ws, rank)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2009_07226_b200 import _lib, geometry, pipeline, solver

    from paper_2009_07226_b200 import parallel
    scfg = pipeline.SystemConfig(precision=cfg["precision"], ffactor=16, order=args.order)
    # slices on this rank: weak scaling = a fixed group per GPU; strong
    # scaling = the config's total split by the reference's P_b rule
    domain = args.partition == "domain" and ws > 1
    cfg["domain"] = domain
    if domain:
        cfg["strong"] = True          # the same problem, split by image/sinogram tiles
        S = cfg["slices"]
    elif cfg.get("strong"):
        lo, hi = parallel.slice_groups(cfg["slices"], ws)[rank]
        S = hi - lo
    else:
        S = cfg["slices"]
    t0 = time.perf_counter()
    system, t_matrix = None, 0.0
    if rank == 0:
        g, y1 = make_problem(cfg, S)
        t_matrix = time.perf_counter() - t0
        if not domain:
            system = pipeline.assemble(g, scfg)
        geometry.clear_matrix_cache()
        torch.cuda.empty_cache()
    else:
        g = geometry.make_geometry(cfg["k"], S, cfg["n"])
    if domain:
        import dataclasses
        scfg = dataclasses.replace(scfg, p_d=ws)
        system = parallel.DomainPartitionedSystem(g, scfg)
        yt = (torch.from_numpy(y1).to(dev) if rank == 0 else
              torch.empty((g.num_rays, 1), dtype=torch.float64, device=dev))
        dist.broadcast(yt, src=0)
        y1 = yt.cpu().numpy()
    elif ws > 1:
        # one host build; the staged operator goes to every GPU over NVLink
        system = parallel.broadcast_system(system, scfg, g)
        yt = (torch.from_numpy(y1).to(dev) if rank == 0 else
              torch.empty((g.num_rays, 1), dtype=torch.float64, device=dev))
        dist.broadcast(yt, src=0)
        y1 = yt.cpu().numpy()
    y = np.broadcast_to(y1, (g.num_rays, S))      # identical phantom slices
    torch.cuda.synchronize()
    t_assemble = time.perf_counter() - t0 - t_matrix
    nnz = system.matrix.nnz if not domain else int(round(_global_nnz(system)))

    W, K = max(args.warmup, 0), max(args.steps, 1)
    run = solver.CGLSRun(system, y, solver.SolveConfig(max_iters=W + K + 1,
                                                       precision=cfg["precision"]))
    run.start()
    for _ in range(W):
        run.step()
    events = []
    run.cg.events = events
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record()
        for _ in range(K):
            run.step()
        e1.record()
        torch.cuda.synchronize()
    launches = _lib.launch_count[0] - launches0
    run.cg.events = None
    if ws > 1:
        dist.barrier()
    t_local = e0.elapsed_time(e1) / 1e3
    t_max = t_local
    if ws > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    t_iter = t_max / K
    flops_iter = 4.0 * nnz * S            # forward + adjoint, 2 flops per nnz per slice
    S_total = cfg["slices"] if cfg.get("strong") else cfg["slices"] * ws
    value = 4.0 * nnz * S_total / t_iter / 1e9

    # roofline of the staged SpMM (compulsory bytes)
    from paper_2009_07226_b200 import matrixstore
    b_e = 2 + matrixstore.element_bytes(cfg["precision"])
    b_x = matrixstore.element_bytes(cfg["precision"])
    n_chunks = -(-S // 16)
    R, C = g.num_rays, g.num_voxels

    def side_bytes(side):       # compulsory bytes of one launch on this rank
        blk = side.blocks[0]
        return blk.nnz * b_e * n_chunks + (blk.n_in + blk.n_out) * S * b_x
    bytes_fwd, bytes_adj = side_bytes(system.forward), side_bytes(system.adjoint)
    bytes_app = (bytes_fwd + bytes_adj) / 2
    # events: (forward?, start, end[, fraction of the application]) -- the
    # domain-partitioned operator launches K6 in F-chunk waves
    spmm_ms = [e[1].elapsed_time(e[2]) for e in events]
    t_spmm = sum(spmm_ms) / 1e3
    frac = [e[3] if len(e) > 3 else 1.0 for e in events]
    n_spmm = sum(frac)
    moved = sum((bytes_fwd if e[0] else bytes_adj) * f for e, f in zip(events, frac))
    achieved = moved / t_spmm / 1e9 if t_spmm > 0 else 0.0
    peak, peak_src = hbm_peak()
    local_nnz = (system.forward.blocks[0].nnz + system.adjoint.blocks[0].nnz) / 2
    spmm_gflops = 2.0 * local_nnz * S * n_spmm / t_spmm / 1e9 if t_spmm > 0 else 0.0
    traffic = None
    tf = ROOT / "profiles" / f"traffic_{args.config}_{cfg['precision']}.json"
    if tf.exists() and ws == 1:     # the ncu capture is of the one-GPU launch
        traffic = json.loads(tf.read_text()).get("bytes_per_launch")

    # end to end through the public API: host y in (pinned), host x out
    e2e = None
    if not args.no_e2e:
        iters = args.e2e_iters or min(cfg["iters"], 10)
        y_host = torch.from_numpy(np.ascontiguousarray(y)).pin_memory()
        del run
        torch.cuda.empty_cache()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = solver.cgls_solve(system, y_host, solver.SolveConfig(max_iters=iters,
                                                                   precision=cfg["precision"]))
        x_host = res.x
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - t0
        if ws > 1:
            tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": 4.0 * nnz * S_total * res.iterations / t_e2e / 1e9, "unit": "GFLOPS",
               "h2d_bytes_per_step": int(y_host.numel() * 8),
               "d2h_bytes_per_step": int(x_host.numel() * 8),
               "step": f"one cgls_solve({iters} iterations) call with host arrays",
               "s_per_call": t_e2e, "iterations": res.iterations}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        r = cpu_baseline(cfg, S)
        cpu_gflops = flops_iter / r["t_iter_extrap"] / 1e9
        cpu = {"value": cpu_gflops, "unit": "GFLOPS", "cores": 1, "kind": "port",
               "sample": f"oracle port, views 0..{r['kp'] - 1} of {cfg['k']} (bit-exact angle "
                         f"subset), {r['sp']} of {S} slices, one CGLS iteration "
                         f"({r['t_iter_sample']:.2f} s), extrapolated x{r['scale']:.0f}",
               "cg_s_per_iter": r["t_iter_extrap"]}

    if rank == 0:
        line = {
            "metric": metric_name(cfg), "value": value, "unit": "GFLOPS", "n_gpus": ws,
            "steps": K, "warmup": W, "ms_per_step": t_iter * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None,
            "dtype": "f32" if cfg["precision"] == "single" else
                     ("f16 storage / f32 accumulate" if cfg["precision"] == "mixed"
                      else cfg["precision"]),
            "data": "synthetic Shepp-Logan phantom, y = A x (float64, on device)",
            "config": config_block(cfg, ws),
            "cg_s_per_iter": t_iter, "voxels_per_s": C * S_total / t_iter,
            "spmm_gflops_kernel": spmm_gflops, "spmm_launches_timed": n_spmm,
            "nnz": nnz, "assemble_s": t_assemble, "matrix_build_s": t_matrix,
            "operator_hbm_bytes": system.hbm_bytes(),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_src,
                         "bytes_per_launch": bytes_app,
                         "bytes_model": "nnz*(2+b_x)*ceil(S/16) + (rays+voxels)*S*b_x"},
            "clocks": clocks.summary(),
            "gpu_launches": launches,
            "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
