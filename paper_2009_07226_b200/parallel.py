"""Multi-GPU plumbing: one process per GPU, torch.distributed over NCCL.

Slice-batch parallelism (P_b, src/cli.py:158-200): the slices are split
into contiguous groups (first S mod P_b groups get one more) and every GPU
runs an independent CGLS on its group with its own alpha/beta -- no
data-path collective.  Every GPU needs the whole operator; it is built once
on the source rank and broadcast over NVLink (NCCL) instead of being rebuilt
per rank, so host memory and build time do not scale with the GPU count.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import matrixstore, pipeline

__all__ = ["slice_groups", "broadcast_system", "MatrixInfo"]


def slice_groups(num_slices: int, p_b: int) -> list:
    """Contiguous batch groups, first S%P_b get +1 (src/cli.py:158-168)."""
    base, rem = divmod(num_slices, p_b)
    out, start = [], 0
    for i in range(p_b):
        size = base + (1 if i < rem else 0)
        if size == 0:
            continue
        out.append((start, start + size))
        start += size
    return out


@dataclass
class MatrixInfo:
    """What an operator on a non-building rank knows about the matrix."""

    num_rows: int
    num_cols: int
    nnz: int
    num_angles: int
    num_detector_cols: int


def _bcast_side(side, src, rank, dev):
    import torch
    import torch.distributed as dist
    meta = [matrixstore.side_meta(side) if rank == src else None]
    dist.broadcast_object_list(meta, src=src, device=dev)
    meta = meta[0]
    tensors = {}
    for k, (shape, dtype) in meta["tensors"].items():
        if rank == src:
            t = side.tensors[k]
        else:
            t = torch.empty(shape, dtype=getattr(torch, dtype), device=dev)
        # raw bytes: int16 slot arrays are not an NCCL/gloo dtype
        dist.broadcast(t.view(-1).view(torch.uint8), src=src)
        tensors[k] = t
    if rank == src:
        return side
    return matrixstore.side_from_meta(meta, tensors)


def broadcast_system(system, config, geometry, src: int = 0):
    """Return the rank-local AssembledSystem, built on `src` only (P_d = 1)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank()
    dev = torch.device("cuda", torch.cuda.current_device())
    if rank == src and (len(system.forward.blocks) != 1 or
                        system.forward.input_elements[0] is not None):
        raise ValueError("broadcast_system supports the single-block (P_d = 1) operator")
    meta = [None]
    if rank == src:
        m = system.matrix
        meta = [dict(num_rows=int(m.num_rows), num_cols=int(m.num_cols), nnz=int(m.nnz),
                     num_angles=int(getattr(m, "num_angles", m.num_rows)),
                     num_detector_cols=int(getattr(m, "num_detector_cols", 1)),
                     exp=int(system.value_scale_exp))]
    dist.broadcast_object_list(meta, src=src, device=dev)
    meta = meta[0]
    fwd = _bcast_side(system.forward.blocks[0] if rank == src else None, src, rank, dev)
    adj = _bcast_side(system.adjoint.blocks[0] if rank == src else None, src, rank, dev)
    if rank == src:
        return system
    info = MatrixInfo(meta["num_rows"], meta["num_cols"], meta["nnz"], meta["num_angles"],
                      meta["num_detector_cols"])
    return pipeline.AssembledSystem.from_sides(info, config, geometry, fwd, adj, meta["exp"])
