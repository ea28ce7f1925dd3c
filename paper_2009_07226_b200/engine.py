"""Kernel launch layer of the staged SpMM (K6) and the reference-compatible
engine surface (src/engine.py): Minibatch, PartialResult, KernelCounters,
flops_and_bytes, spmm_reference, MAX_FFACTOR.

``apply_side`` is the single entry into ``xct_spmm``: every forward and back
projection of the pipeline and of CGLS goes through it.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .matrixstore import DeviceSide, element_bytes, storage_dtype

__all__ = ["MAX_FFACTOR", "Minibatch", "PartialResult", "KernelCounters", "apply_side",
           "spmm_reference", "csr_spmm_f64", "flops_and_bytes", "kernel_counters"]

MAX_FFACTOR = 50          # src/engine.py:38


@dataclass
class Minibatch:
    """F fused slice vectors (elements, F) at one precision (src/engine.py:41-61)."""

    data: np.ndarray
    precision: str

    def __post_init__(self):
        if self.data.ndim != 2:
            raise ValueError("minibatch data must be (elements, ffactor)")
        if not 1 <= self.ffactor <= MAX_FFACTOR:
            raise ValueError(f"fusing factor must be in [1, {MAX_FFACTOR}]")

    @property
    def ffactor(self) -> int:
        return self.data.shape[1]

    @staticmethod
    def from_columns(data: np.ndarray, precision: str) -> "Minibatch":
        return Minibatch(np.ascontiguousarray(data, dtype=storage_dtype(precision)), precision)


@dataclass
class PartialResult:
    """One process's partial output over its footprint (src/engine.py:64-75)."""

    owner: int
    elements: np.ndarray = field(repr=False)
    values: np.ndarray = field(repr=False)
    precision: str = "double"

    @property
    def ffactor(self) -> int:
        return self.values.shape[1]


# tuning override of the chunk-group schedule (tools/spmm_probe.py sweeps)
_TUNE_GROUP = int(os.environ["XCT_SPMM_CHUNK_GROUP"]) if os.environ.get("XCT_SPMM_CHUNK_GROUP") else None


def apply_side(side: DeviceSide, x_chunked, out, *, row_stride: int, chunk_stride: int,
               valid_cols: int, ffactor_out: int, factors=None, dot_partials=None,
               stream=None, x_chunk_stride: int = 0, x_elem_stride: int = 0,
               out_ptrs=None, seg=None) -> None:
    """Launch K6 on one staged side.

    x_chunked: device tensor [n_chunks, n_in, f_dev] at the storage dtype
         (or any layout given by x_chunk_stride / x_elem_stride in records,
         e.g. [n_in, n_chunks, f_dev]: x_chunk_stride=1, x_elem_stride=n_chunks).
    out: device f32 (f64 in double) tensor addressed as
         out[row*row_stride + chunk*chunk_stride + j], j < ffactor_out,
         chunk*ffactor_out + j < valid_cols.
    factors: f64 [n_chunks] denormalize factors; dot_partials: f64
         [n_chunks * n_cta] receives per-CTA sums of squares of the outputs.
    """
    n_chunks = int(x_chunked.shape[1] if x_elem_stride else x_chunked.shape[0])
    ep = _lib.Epilogue()
    ep.d_out = out.data_ptr() if out is not None else None
    ep.row_stride, ep.chunk_stride = int(row_stride), int(chunk_stride)
    ep.valid_cols, ep.ffactor = int(valid_cols), int(ffactor_out)
    ep.value_scale_exp = int(side.value_scale_exp)
    ep.accumulate = 0
    ep.d_factors = None if factors is None else factors.data_ptr()
    ep.d_dot_partials = None if dot_partials is None else dot_partials.data_ptr()
    ep.x_chunk_stride, ep.x_elem_stride = int(x_chunk_stride), int(x_elem_stride)
    if out_ptrs is not None:       # fused exchange: rows scattered by segment
        ep.d_out_ptrs, ep.d_seg, ep.n_seg = out_ptrs.data_ptr(), seg.data_ptr(), out_ptrs.numel()
    st = stream if stream is not None else _lib.stream_handle(x_chunked.device)
    if _TUNE_GROUP is not None:
        side.staged.chunk_group = _TUNE_GROUP
    _lib.check(_lib.lib().xct_spmm(C.byref(side.staged), _lib.PREC_CODE[side.precision],
                                   x_chunked.data_ptr(), side.n_in, n_chunks, side.f_dev,
                                   C.byref(ep), side.smem_bytes, st), "xct_spmm")
    _lib.count_launches("xct_spmm")


def apply_side_ptr(side: DeviceSide, x_ptr: int, n_chunks: int, out, **kw) -> None:
    """apply_side on an input given as a raw device pointer (e.g. a CUDA IPC
    receive buffer) of n_chunks F-chunks; layout by the x_* strides."""
    class _X:                                   # the two attributes apply_side reads
        shape = (side.n_in, n_chunks) if kw.get("x_elem_stride") else (n_chunks, side.n_in)
        device = out.device

        @staticmethod
        def data_ptr():
            return int(x_ptr)
    apply_side(side, _X, out, **kw)


def csr_spmm_f64(matrix, x: np.ndarray) -> np.ndarray:
    """y = A x in float64 on the device for a canonical CSR (host x)."""
    import torch
    from .geometry import device
    dev = device()
    X = np.ascontiguousarray(x.reshape(x.shape[0], -1), np.float64)
    d_x = torch.from_numpy(X).to(dev)
    ip = getattr(matrix, "d_indptr", None)
    if ip is None:
        ip = torch.as_tensor(np.asarray(matrix.indptr, np.int64), device=dev)
        ix = torch.as_tensor(np.asarray(matrix.indices, np.int32), device=dev)
        vv = torch.as_tensor(np.asarray(matrix.values, np.float64), device=dev)
    else:
        ix, vv = matrix.d_indices, matrix.d_values
    n_rows = int(ip.numel()) - 1
    y = torch.empty((n_rows, X.shape[1]), dtype=torch.float64, device=dev)
    _lib.call("xct_csr_spmm_f64", ip.data_ptr(), ix.data_ptr() if ix.numel() else None,
              vv.data_ptr() if vv.numel() else None, n_rows, d_x.data_ptr(), X.shape[1],
              y.data_ptr(), _lib.stream_handle(dev))
    out = y.cpu().numpy()
    return out.reshape(n_rows) if x.ndim == 1 else out


def spmm_reference(block, x: np.ndarray) -> np.ndarray:
    """Double-precision product of any compressed-row operator (the
    reference's FP64 ground truth, src/engine.py:78-101), on the device."""
    cols = x.reshape(-1, 1) if x.ndim == 1 else x
    if cols.shape[0] != block.num_cols:
        raise ValueError(f"input has {cols.shape[0]} elements, block expects {block.num_cols}")
    out = csr_spmm_f64(block, cols)
    return out[:, 0] if x.ndim == 1 else out


@dataclass
class KernelCounters:
    """Work/traffic of one application (src/engine.py:224-242)."""

    nnz: int
    ffactor: int
    precision: str
    flops: int
    entry_bytes: int
    gather_bytes: int
    output_bytes: int

    @property
    def total_bytes(self) -> int:
        return self.entry_bytes + self.gather_bytes + self.output_bytes

    @property
    def arithmetic_intensity(self) -> float:
        return self.flops / self.total_bytes if self.total_bytes else 0.0


def flops_and_bytes(side: DeviceSide, ffactor: int | None = None,
                    precision: str | None = None) -> KernelCounters:
    """2 flops per entry per slice; padded entry bytes, staged gathers and
    outputs of the B200 format (src/engine.py:245-261)."""
    ff = ffactor or side.ffactor
    prec = precision or side.precision
    eb = element_bytes(prec)
    return KernelCounters(nnz=side.nnz, ffactor=ff, precision=prec, flops=2 * side.nnz * ff,
                          entry_bytes=side.padded_entries * (2 + eb),
                          gather_bytes=int(side.info.n_slots) * eb * ff,
                          output_bytes=side.n_out * eb * ff)


def kernel_counters(sides) -> KernelCounters:
    total = None
    for s in sides:
        c = flops_and_bytes(s)
        if total is None:
            total = c
        else:
            total = KernelCounters(total.nnz + c.nnz, c.ffactor, c.precision,
                                   total.flops + c.flops, total.entry_bytes + c.entry_bytes,
                                   total.gather_bytes + c.gather_bytes,
                                   total.output_bytes + c.output_bytes)
    return total
