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

Default workload: BASELINE.json's metric shape, config c5 (2048^2 image,
2048 views, 1024 slices, FP16 storage with FP32 accumulation) on one GPU.
The line also carries in-run checks tying the number to a verified result:
adjointness <A x, y> = <x, A^T y> of the timed fast path on one F-chunk,
a non-increasing residual, and the FP16 residual curve against an FP32 CGLS
on a 16-slice subset run through an independent matrix-free FP32 Siddon
operator (K11).

Multi-GPU (torchrun): slice-batch partitioning P_b = N (src/cli.py:158-200)
by default -- each rank reconstructs its own slice group of the same
geometry, no data-path collective -- or image-domain tiles with the NCCL
partial-result exchange (--partition domain); timing is max over ranks.

  python bench.py [--config c5] [--steps K] [--warmup W] [--impl b200|reference]
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


# CPU sample of the workload (BASELINE.md / SURVEY.md §8(d)(ii)): K' views
# spread evenly over [0, pi) are bit-identical to every (K/K')-th view of
# the full geometry when K/K' is a power of two (angles = i * pi / K), so the
# sample's entries per view are representative of the whole operator.
SAMPLE_VIEWS, SAMPLE_SLICES = 8, 16


def _cpu_sample(cfg, sample_views=SAMPLE_VIEWS, sample_slices=SAMPLE_SLICES):
    """Oracle port of the reference CPU path (oracle/xct_oracle.py, the
    restatement of src/pipeline.py + src/solver.py) on the view/slice
    sample: Shepp-Logan y = A x (src/geometry.py:327-367) and the staged
    operator (the reference's assembly, untimed)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import xct_oracle as O
    K, N = cfg["k"], cfg["n"]
    kp, sp = min(sample_views, K), sample_slices
    if K % kp or (K // kp) & (K // kp - 1):
        if K * N > 1 << 16:
            raise ValueError("the view sample must divide K by a power of two")
        kp = K                      # small configs (c1): the whole view set, no extrapolation
    g = O.make_geom(kp, sp, N)
    A = O.system_matrix(g)
    y = O.measure(A, O.phantom("shepp-logan-like", N, sp))
    op = O.Operator(A, g, cfg["precision"], 16)
    op.adjoint(y.astype(np.float32))          # staging tables built (= assembly), untimed
    op.forward(np.zeros((A.num_cols, sp), np.float32))
    return O, op, y, dict(kp=kp, sp=sp, nnz_sample=A.nnz, scale=(K / kp))


def _extrap_label(factor: float) -> str:
    return "the whole workload, not extrapolated" if factor <= 1.0 else \
        f"EXTRAPOLATED x{factor:.0f}"


def cpu_baseline(cfg, slices, iters=2):
    """One host core: the oracle's CGLS iterations (projection, back
    projection, dots, normalize/store -- the whole reference iteration,
    src/solver.py:160-192) on the sample; per-iteration time extrapolated
    by (K/K') views x (S/S') slices."""
    O, op, y, info = _cpu_sample(cfg)
    r = O.cgls(op, y, iters, cfg["precision"])
    t = statistics.median(r["iteration_seconds"])
    info.update(t_iter_sample=t, iters=len(r["iteration_seconds"]),
                t_iter_extrap=t * info["scale"] * (slices / info["sp"]))
    return info


def _reference_worker(job):
    """One host core's share of the reference arm: build the sample once,
    then time `n` CGLS iterations of it."""
    cfg, n = job
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    if n == 0:
        return None
    O, op, y, info = _cpu_sample(cfg)
    r = O.cgls(op, y, n, cfg["precision"])
    info["times"] = r["iteration_seconds"]
    return info


def run_reference_arm(args, cfg, ws, rank):
    """--impl reference: the reference CPU path (the oracle port of
    src/engine.py + src/solver.py; the reference is pure Python with no
    build, so there is no oracle/_ref) on every host core.  The reference
    solves slice groups independently (P_b, src/cli.py:158-200), so each
    core runs its own sample problem; the W + K step iterations are spread
    over the cores (each core times its share after building its sample),
    and the cores' iteration rates add up.  Per-step work: one CGLS
    iteration over the view/slice sample, extrapolated to the full
    workload."""
    if rank != 0:
        return
    import multiprocessing as mp
    total = cfg["slices"] if cfg.get("strong") else cfg["slices"] * ws
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    n = args.warmup + args.steps
    per = [n // cores + (1 if i < n % cores else 0) for i in range(cores)]
    per = [max(1, p) for p in per]                     # every core does work
    with mp.get_context("fork").Pool(cores) as pool:
        runs = pool.map(_reference_worker, [(cfg, p) for p in per])
    info = runs[0]
    # a core's iterations after the first are steady state (the first of
    # each core pays cold caches); cores ran concurrently
    t_core = [statistics.median(r["times"][1:] if len(r["times"]) > 1 else r["times"])
              for r in runs]
    t_sample = 1.0 / sum(1.0 / t for t in t_core)      # all cores together
    t = t_sample * info["scale"] * (total / info["sp"])
    nnz_full = info["nnz_sample"] * info["scale"]
    gflops = 4.0 * nnz_full * total / t / 1e9
    line = {"impl": "reference", "metric": metric_name(cfg), "value": gflops, "unit": "GFLOPS",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg.get("strong") else "weak",
            "vs_baseline": None, "dtype": "f32" if cfg["precision"] == "single" else "f16/f32",
            "data": "synthetic", "config": config_block(cfg, ws),
            "cg_s_per_iter": t,
            "cpu_baseline": {"value": gflops, "unit": "GFLOPS", "cores": cores, "kind": "port",
                             "sample": f"oracle port on {cores} host cores (one sample problem "
                                       f"per core, {sum(per)} CGLS iterations spread over them, "
                                       f"the first of each core untimed when it ran more): "
                                       f"{info['kp']} of {cfg['k']} views (every "
                                       f"{cfg['k'] // info['kp']}th, bit-exact), "
                                       f"{info['sp']} of {total} slices; "
                                       + _extrap_label(info['scale'] * total / info['sp']),
                             "per_core_s_per_iter_sample": t_core},
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


def _fp32_reference_curve(g, y16, iters):
    """CGLS in FP32 with the reference's scalar/cast sequence (f64 dots,
    alpha/beta cast to f32, multiply-then-add updates; src/solver.py:129-196)
    over the independent matrix-free FP32 operator (K11).  Verification
    only: the vector updates are plain torch ops."""
    import torch
    from paper_2009_07226_b200 import geometry
    A = lambda v: geometry.project_matrix_free_f32(g, v)
    At = lambda v: geometry.project_matrix_free_f32(g, v, adjoint=True)
    dot = lambda a, b: float(torch.sum(a.double() * b.double()))
    Y = y16.double()
    ynorm = math.sqrt(dot(Y, Y))
    x = torch.zeros((g.num_voxels, 16), dtype=torch.float32, device=y16.device)
    r = y16.clone()
    s = At(r)
    p = s.clone()
    gam = gam0 = dot(s, s)
    curve = []
    for _ in range(iters):
        q = A(p)
        al = np.float32(gam / dot(q, q))
        x = x + (p * float(al))
        r = r - (q * float(al))
        s = At(r)
        gn = dot(s, s)
        be = np.float32(gn / gam)
        gam = gn
        p = s + (p * float(be))
        curve.append(math.sqrt(dot(r, r)) / ynorm)
    return curve, gam0


def run_checks(args, cfg, g, system, y1, history, dev):
    """Full-size checks of the timed fast path:
    adjointness on one F-chunk, a non-increasing residual over the timed
    run, and the residual curve against FP32 on a 16-slice subset (every
    phantom slice is identical, so the subset's curve is the run's)."""
    import torch
    out = {}
    t0 = time.perf_counter()
    gen = torch.Generator(device=dev).manual_seed(1)
    xr = torch.rand((g.num_voxels, 16), generator=gen, device=dev, dtype=torch.float32)
    yr = torch.rand((g.num_rays, 16), generator=gen, device=dev, dtype=torch.float32)
    ax, _ = system.apply_forward(xr)
    aty, _ = system.apply_adjoint(yr)
    lhs = float(torch.sum(ax.double() * yr.double()))
    rhs = float(torch.sum(xr.double() * aty.double()))
    # the same projection through the independent FP32 operator
    from paper_2009_07226_b200 import geometry
    ax32 = geometry.project_matrix_free_f32(g, xr)
    fwd_rel = float(torch.linalg.vector_norm((ax - ax32).double()) /
                    torch.linalg.vector_norm(ax32.double()))
    del ax, aty, ax32
    tol_adj = 2e-3 if cfg["precision"] in ("half", "mixed") else 1e-5
    out["adjointness"] = {"lhs": lhs, "rhs": rhs, "rel_diff": abs(lhs - rhs) / abs(rhs),
                          "tol": tol_adj, "ok": abs(lhs - rhs) <= tol_adj * abs(rhs),
                          "what": "<A x, y> vs <x, A^T y>, random x, y in [0,1), one F-chunk "
                                  "of 16 slices, timed precision and order"}
    tol_fwd = 2e-3 if cfg["precision"] in ("half", "mixed") else 1e-5
    out["forward_vs_fp32_matrix_free"] = {"rel_l2": fwd_rel, "tol": tol_fwd,
                                          "ok": fwd_rel <= tol_fwd}
    h = np.asarray(history)
    worst = float(np.max(h[1:] / h[:-1] - 1.0)) if len(h) > 1 else 0.0
    out["residual_monotone"] = {"iterations": len(h), "max_rel_increase": worst,
                                "tol": 1e-3, "ok": worst <= 1e-3,
                                "first": float(h[0]) if len(h) else None,
                                "last": float(h[-1]) if len(h) else None}
    n = min(args.check_iters, len(h))
    if n:
        y16 = torch.from_numpy(np.ascontiguousarray(y1, np.float32)).to(dev).expand(
            g.num_rays, 16).contiguous()
        ref, _ = _fp32_reference_curve(g, y16, n)
        ratio = h[:n] / np.asarray(ref)
        lead = int(np.argmax(np.abs(ratio - 1.0) > 0.02)) if np.any(np.abs(ratio - 1.0) > 0.02) \
            else n
        # FP16 storage tracks FP32 until its quantization floor, then sits
        # above it: the reference's own mixed/single residual ratio reaches
        # 1.36 at config 1 and 1.23 at N = K = 256 (tests/golden: c1,
        # sub256) and its test bounds it by 3 (tests/test_solver.py:137-148);
        # the check bounds it by 1.5 at every iteration
        out["residual_curve_vs_fp32"] = {
            "iterations": n, "slices": 16, "fp32_curve": [float(v) for v in ref],
            "run_curve": [float(v) for v in h[:n]],
            "max_ratio": float(ratio.max()), "min_ratio": float(ratio.min()),
            "leading_iterations_within_2pct": lead, "tol_ratio": 1.5,
            "ok": bool(ratio.max() <= 1.5 and ratio.min() >= 1.0 / 1.5),
            "fp32_operator": "matrix-free Siddon, FP32 (K11 xct_siddon_project_f32)"}
    out["seconds"] = time.perf_counter() - t0
    out["ok"] = all(v.get("ok", True) for v in out.values() if isinstance(v, dict))
    return out


def measure_exchange(run, system, ws, dev, k6_fwd_s=0.0):
    """NVLink traffic of the domain partition's exchanges: bytes each rank
    sends per application (counted over the run) and the NCCL p2p time of
    one extra CG iteration with the exchange phases serialized
    (XCT_EXCHANGE_PROFILE=1, domain.py) -- GB/s per rank against NVLink 5's
    900 GB/s per direction (nominal) and the pool's measured 770 GB/s peer
    copy (B200_PROFILING.md).  Max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2009_07226_b200 import domain
    bytes_run = {k: v["bytes_out_per_application"] for k, v in system.exchange_stats().items()}
    for side in (system.forward, system.adjoint):
        side.stats = domain._Stats()
    os.environ["XCT_EXCHANGE_PROFILE"] = "1"
    try:
        run.step()
    finally:
        os.environ.pop("XCT_EXCHANGE_PROFILE", None)
    st = system.exchange_stats()
    out = {}
    fused = getattr(system.forward, "fused", False) and ws > 1
    if fused and "projection" in st:
        # fused exchange: the forward's peer rows leave as remote stores from
        # K6's epilogue, overlapping the math; report the bytes and the rate
        # they needed over the K6 time
        v = st.pop("projection")
        t = torch.tensor([bytes_run.get("projection", v["bytes_out_per_application"]),
                          k6_fwd_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["projection"] = {"mode": "fused: K6 epilogue stores into peers' receive buffers "
                                     "(CUDA IPC over NVLink), no separate transfer phase",
                             "bytes_out_per_rank_max": float(t[0]),
                             "k6_forward_ms_max": float(t[1]) * 1e3,
                             "gbs_per_rank_during_k6": float(t[0]) / float(t[1]) / 1e9
                             if float(t[1]) > 0 else None,
                             "payload": "f32 partials"}
    for name, v in st.items():
        t = torch.tensor([v["nccl_seconds_per_application"],
                          bytes_run.get(name, v["bytes_out_per_application"])],
                         dtype=torch.float64, device=dev)
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum)
        sec, byt = float(tmax[0]), float(tmax[1])
        gbs = byt / sec / 1e9 if sec > 0 else 0.0
        out[name] = {"mode": ("fused: the owners' gather kernels store into the consumers' "
                              "K6 inputs over NVLink (CUDA IPC); time = that phase, "
                              "barriers included") if fused else "NCCL p2p, F-chunk waves",
                     "bytes_out_per_rank_max": byt, "bytes_total": float(tsum[1]),
                     "nccl_ms_max": sec * 1e3, "gbs_per_rank": gbs,
                     "frac_of_900_nominal": gbs / 900.0, "frac_of_770_measured": gbs / 770.0,
                     "payload": "f32 partials" if name == "projection" else
                                "normalized inputs at the storage dtype"}
    out["note"] = ("times of one extra CG iteration with the exchange phases serialized "
                   "(XCT_EXCHANGE_PROFILE=1); " + ("fused mode (default): the projection's "
                   "transfer is inside K6" if fused else
                   f"the timed run overlaps the NCCL p2p with K6 in {domain._Waves.WAVES} "
                   "F-chunk waves"))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--no-checks", action="store_true")
    ap.add_argument("--check-iters", type=int, default=30)
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

    from paper_2009_07226_b200 import matrixstore, parallel
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
    g = geometry.make_geometry(cfg["k"], S, cfg["n"])
    # slice batch: with the device format build every GPU assembles its own
    # copy of the operator in parallel; otherwise rank 0 builds on the host
    # and broadcasts it over NVLink
    own_build = not domain and (ws == 1 or (
        pipeline._streamable(g, scfg) and
        matrixstore.device_build_supported(pipeline.Plan_probe(scfg), scfg.precision)))
    if rank == 0:
        g, y1 = make_problem(cfg, S)
        t_matrix = time.perf_counter() - t0
        if not domain:
            system = pipeline.assemble(g, scfg)
        geometry.clear_matrix_cache()
        torch.cuda.empty_cache()
    elif own_build:
        system = pipeline.assemble(g, scfg)
        torch.cuda.empty_cache()
    if domain:
        import dataclasses
        scfg = dataclasses.replace(scfg, p_d=ws)
        system = parallel.DomainPartitionedSystem(g, scfg)
        yt = (torch.from_numpy(y1).to(dev) if rank == 0 else
              torch.empty((g.num_rays, 1), dtype=torch.float64, device=dev))
        dist.broadcast(yt, src=0)
        y1 = yt.cpu().numpy()
    elif ws > 1:
        if not own_build:
            # one host build; the staged operator goes to every GPU over NVLink
            system = parallel.broadcast_system(system, scfg, g)
        yt = (torch.from_numpy(y1).to(dev) if rank == 0 else
              torch.empty((g.num_rays, 1), dtype=torch.float64, device=dev))
        dist.broadcast(yt, src=0)
        y1 = yt.cpu().numpy()
    # identical phantom slices: a zero-stride device view, streamed into the
    # solver one block of rows at a time (no (rays, S) float64 copy anywhere)
    y_dev = torch.from_numpy(np.ascontiguousarray(y1)).to(dev).expand(g.num_rays, S)
    torch.cuda.synchronize()
    t_assemble = time.perf_counter() - t0 - t_matrix
    nnz = system.matrix.nnz if not domain else int(round(_global_nnz(system)))

    W, K = max(args.warmup, 0), max(args.steps, 1)
    run = solver.CGLSRun(system, y_dev, solver.SolveConfig(max_iters=W + K + 1,
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

    history = list(run.result.residual_history)
    exchange = None
    if domain and getattr(system, "native", False):
        fwd = [e[1].elapsed_time(e[2]) / 1e3 for e in events if e[0]]
        exchange = measure_exchange(run, system, ws, dev,
                                    sum(fwd) / max(1, sum(1 for e in events if e[0])))
    del run
    torch.cuda.empty_cache()

    # in-run checks of the timed configuration (rank 0's operator)
    checks = None
    if not args.no_checks and not domain:
        checks = run_checks(args, cfg, g, system, y1, history, dev)

    # end to end through the public API: host float32 y in (pinned), host
    # float64 x out (src/solver.py:129-196), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        iters = args.e2e_iters or min(cfg["iters"], 10)
        n_loc = getattr(system, "local_rows", g.num_rays) if domain else g.num_rays
        y_host = torch.empty((g.num_rays, S), dtype=torch.float32, pin_memory=True)
        y_host.copy_(torch.from_numpy(y1.astype(np.float32)).expand(g.num_rays, S))
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
               "h2d_bytes_per_step": int(n_loc * S * 4),
               "d2h_bytes_per_step": int(x_host.numel() * 8),
               "step": f"one cgls_solve({iters} iterations) call: pinned host float32 y "
                       f"in, host float64 x out",
               "s_per_call": t_e2e, "iterations": res.iterations}
        del x_host, res, y_host

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:      # N = 1 only
        r = cpu_baseline(cfg, S)
        cpu_gflops = flops_iter / r["t_iter_extrap"] / 1e9
        cpu = {"value": cpu_gflops, "unit": "GFLOPS", "cores": 1, "kind": "port",
               "sample": f"oracle port on 1 core: {r['iters']} CGLS iterations over "
                         f"{r['kp']} of {cfg['k']} views (every {cfg['k'] // r['kp']}th, "
                         f"bit-exact) x {r['sp']} of {S} slices, {r['t_iter_sample']:.2f} s "
                         f"per iteration; " + _extrap_label(r['scale'] * S / r['sp']),
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
            "e2e": e2e, "cpu_baseline": cpu, "checks": checks,
        }
        if exchange is not None:
            line["nvlink_exchange"] = exchange
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
