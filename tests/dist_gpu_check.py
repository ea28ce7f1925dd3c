"""Multi-GPU check of the data-partitioned operator (run under torchrun on
>= 2 GPUs; driven by tests/test_gpu_multi.py).  Compares the NCCL operator
with the one-process emulation of the same partition (bit-exact in
reference order) and with the single-GPU native operator (tolerance)."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2009_07226_b200 import geometry, parallel, pipeline, solver  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main(out_path, n=64, k=96, slices=5):
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    g = geometry.make_geometry(k, slices, n)
    rng = np.random.default_rng(11)
    y = rng.random((g.num_rays, slices))
    report = {}
    for prec in ("single", "mixed"):
        for order in ("reference", "native"):
            cfg = pipeline.SystemConfig(precision=prec, ffactor=4, p_d=ws, order=order,
                                        comm_strategy="direct")
            dps = parallel.DomainPartitionedSystem(g, cfg)
            res = solver.cgls_solve(dps, y, solver.SolveConfig(max_iters=6, precision=prec))
            x = dps.gather_x(res.x)
            if rank == 0:
                emu = pipeline.assemble(g, cfg)        # one-process emulation, same partition
                ref = solver.cgls_solve(emu, y, solver.SolveConfig(max_iters=6, precision=prec))
                one = pipeline.assemble(g, pipeline.SystemConfig(precision=prec, ffactor=4))
                ref1 = solver.cgls_solve(one, y, solver.SolveConfig(max_iters=6, precision=prec))
                import xct_oracle as O
                og = O.make_geom(k, slices, n)
                ora = O.cgls(O.Operator(O.system_matrix(og), og, prec, 4, p_d=ws), y, 6, prec)
                if prec == "single" and order == "reference":
                    from dataclasses import asdict
                    vr, ve = dps.volume_reports(), emu.volume_reports()
                    report["volume_reports_equal"] = all(
                        asdict(vr[s]) == asdict(ve[s]) for s in ("projection", "backprojection"))
                report[f"{prec}_{order}"] = dict(
                    vs_oracle=rel(x, ora["x"]),
                    vs_emulation=rel(x, ref.x), equal_emulation=bool(np.array_equal(x, ref.x)),
                    vs_single_gpu=rel(x, ref1.x),
                    residual=[float(a) for a in res.residual_history],
                    residual_emu=[float(a) for a in ref.residual_history])
    # streamed per-rank build == source-rank build (same tiles, same groups)
    for prec in ("single", "mixed"):
        xs = []
        for build in ("monolithic", "streamed"):
            pipeline.StreamedAssembly.CHUNK_NNZ = 3e5
            pipeline.StreamedAssembly.BAND_NNZ = 2e5
            cfg = pipeline.SystemConfig(precision=prec, ffactor=4, p_d=ws, build=build)
            dps = parallel.DomainPartitionedSystem(g, cfg)
            res = solver.cgls_solve(dps, y, solver.SolveConfig(max_iters=4, precision=prec))
            xs.append(dps.gather_x(res.x))
        if rank == 0:
            report[f"{prec}_streamed_equal"] = dict(equal=bool(np.array_equal(xs[0], xs[1])),
                                                    rel=rel(xs[1], xs[0]))
    # native partition: the fused exchange (K6 epilogue stores into peers'
    # buffers over CUDA IPC) and the NCCL p2p waves give identical results
    for prec in ("single", "mixed"):
        xs = []
        for fused in ("1", "0"):
            os.environ["XCT_FUSED_EXCHANGE"] = fused
            cfg = pipeline.SystemConfig(precision=prec, ffactor=4, p_d=ws)
            dps = parallel.DomainPartitionedSystem(g, cfg)
            assert dps.forward.fused == (fused == "1")
            res = solver.cgls_solve(dps, y, solver.SolveConfig(max_iters=4, precision=prec))
            xs.append(dps.gather_x(res.x))
        os.environ.pop("XCT_FUSED_EXCHANGE")
        if rank == 0:
            report[f"{prec}_fused_equal"] = dict(equal=bool(np.array_equal(xs[0], xs[1])),
                                                 rel=rel(xs[1], xs[0]))
    if rank == 0:
        Path(out_path).write_text(json.dumps(report, indent=1))
        print(json.dumps(report, indent=1))
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
