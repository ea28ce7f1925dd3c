"""ctypes binding of ``libxct_b200.so`` (the C ABI in ``include/xct_b200.h``).

There is no fallback: importing a compute entry point without the built
library, or calling one without a CUDA device, raises.  Device buffers are
torch tensors (plumbing only: allocation, streams); every kernel is ours.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / ("libxct_b200_checked.so" if os.environ.get("XCT_LIB") == "checked"
                     else "libxct_b200.so")

XCT_OK, XCT_EINVAL, XCT_ECUDA, XCT_ESTAGE, XCT_ENOMEM, XCT_ENONFINITE = range(6)
PREC_CODE = {"double": 0, "single": 1, "half": 2, "mixed": 3}

i32, i64, f32, f64, vp = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_void_p


class FormatInfo(C.Structure):
    _fields_ = [("n_cta", i64), ("rows_per_cta", i64), ("rows_per_warp", i64),
                ("warps_per_cta", i64), ("n_groups", i64), ("n_slots", i64),
                ("n_padded", i64), ("nnz", i64), ("max_group_slots", i64),
                ("value_bytes", i32), ("max_rel_quant_error", f64),
                ("underflow_count", i64), ("row_group", i32)]


class Staged(C.Structure):
    _fields_ = [("n_cta", i64), ("rows_per_cta", i64), ("warps_per_cta", i64),
                ("rows_per_warp", i64), ("n_groups", i64),
                ("d_cta_rows", vp), ("d_cta_group_ptr", vp), ("d_group_map_ptr", vp),
                ("d_group_map", vp), ("d_slab_off", vp), ("d_slab_width", vp),
                ("d_slots", vp), ("d_values", vp), ("max_group_slots", i64),
                ("contract", i32), ("chunk_group", i32), ("row_group", i32)]


class FmtdPart(C.Structure):
    _fields_ = [("d_indptr", vp), ("d_indices", vp), ("d_values", vp), ("n_rows", i64),
                ("d_cta_rows", vp), ("d_cta_mode", vp), ("n_cta", i64), ("rows_per_cta", i64),
                ("rows_per_warp", i64), ("base_b", i32), ("n_keys", i32), ("capacity", i32),
                ("sched_rq", i32), ("sched_fast", i32)]


class Epilogue(C.Structure):
    _fields_ = [("d_out", vp), ("row_stride", i64), ("chunk_stride", i64),
                ("valid_cols", i32), ("ffactor", i32), ("value_scale_exp", i32),
                ("accumulate", i32), ("d_factors", vp), ("d_dot_partials", vp),
                ("x_chunk_stride", i64), ("x_elem_stride", i64), ("d_out_ptrs", vp),
                ("d_seg", vp), ("n_seg", i32)]


_SIGS = {
    "xct_abi_version": (i32, []),
    "xct_last_error": (C.c_char_p, []),
    "xct_siddon_count": (i32, [vp, vp, i32, i32, i32, i32, f64, vp, vp]),
    "xct_siddon_fill": (i32, [vp, vp, i32, i32, i32, i32, f64, vp, vp, vp, vp]),
    "xct_siddon_project_f32": (i32, [vp, vp, i32, i32, i32, i32, f64, i32, vp, vp, vp]),
    "xct_csr_filter_cols": (i32, [vp, vp, vp, i64, i32, i32, vp, vp, vp, vp, vp]),
    "xct_csr_filter_map": (i32, [vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp]),
    "xct_format_build": (i32, [i64, i64, vp, vp, vp, i64, i64, i64, vp, vp, vp, i64, i32,
                               i32, i32, i32, i32, i32, C.POINTER(vp)]),
    "xct_format_get_info": (i32, [vp, C.POINTER(FormatInfo)]),
    "xct_format_export": (i32, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "xct_format_free": (None, [vp]),
    "xct_fmtd_scratch_bytes": (i64, []),
    "xct_fmtd_ranges": (i32, [C.POINTER(FmtdPart), vp, vp, vp, vp, vp]),
    "xct_fmtd_count": (i32, [C.POINTER(FmtdPart), vp, vp, i32, vp, vp, vp, vp]),
    "xct_fmtd_fill": (i32, [C.POINTER(FmtdPart), vp, vp, i32, vp, vp, i32, i32, vp, vp, vp, vp,
                            vp, vp, vp, i64, vp, vp, vp]),
    "xct_csr_col_counts": (i32, [vp, vp, i64, i32, i32, vp, vp]),
    "xct_csr_transpose_band": (i32, [vp, vp, vp, i64, i64, i64, i32, i32, vp, vp, vp, vp, vp,
                                     vp]),
    "xct_csr_transpose": (i32, [i64, i64, vp, vp, vp, vp, vp, vp, i32]),
    "xct_spmm": (i32, [C.POINTER(Staged), i32, vp, i64, i64, i32, C.POINTER(Epilogue), i64, vp]),
    "xct_csr_spmm_f64": (i32, [vp, vp, vp, i64, vp, i64, vp, vp]),
    "xct_chunk_maxabs": (i32, [vp, i32, i64, i64, i64, i32, i64, vp, vp]),
    "xct_normalize": (i32, [vp, i32, i64, i64, i64, i32, i64, i32, vp, i32, vp, vp]),
    "xct_dot": (i32, [vp, vp, i32, i64, f32, f32, vp, vp, vp]),
    "xct_sum_f64": (i32, [vp, i64, vp, vp]),
    "xct_maxabs": (i32, [vp, i32, i64, f32, vp, vp]),
    "xct_axpy": (i32, [vp, i32, f32, vp, i32, f32, f64, i64, vp, i32, f32, vp, vp, vp, vp]),
    "xct_chunk_maxabs_chunked": (i32, [vp, i32, f32, i64, i64, i32, vp, vp]),
    "xct_normalize_chunked": (i32, [vp, i32, f32, i64, i64, i32, vp, i32, vp, vp]),
    "xct_unchunk_f64": (i32, [vp, i32, f32, i64, i64, i32, i32, vp, vp]),
    "xct_chunk_from_f64": (i32, [vp, i64, i64, i32, i32, i32, vp, vp]),
    "xct_rows_to_chunked": (i32, [vp, i32, i64, i64, i64, i64, i32, i32, i32, vp, vp, vp, vp,
                                  vp, vp]),
    "xct_unchunk_rows_f64": (i32, [vp, i32, f32, i64, i64, i64, i64, i32, i32, vp, vp]),
    "xct_binade_hist": (i32, [vp, i64, vp, vp]),
    "xct_gather_rows": (i32, [vp, i64, vp, i64, i64, i32, i32, vp, vp]),
    "xct_accumulate_rows": (i32, [vp, i64, vp, vp, i64, i64, i32, i32, vp]),
    "xct_scale_chunks": (i32, [vp, i64, i64, vp, i32, vp, vp, vp]),
    "xct_ipc_alloc": (i32, [i64, C.POINTER(vp), vp]),
    "xct_ipc_open": (i32, [vp, C.POINTER(vp)]),
    "xct_ipc_close": (i32, [vp]),
    "xct_ipc_free": (i32, [vp]),
    "xct_gather_records": (i32, [vp, i64, vp, i64, i64, i64, i32, vp, vp]),
    "xct_accumulate_records": (i32, [vp, i64, i64, vp, vp, i64, i64, i32, i32, vp]),
}

_lib = None


class XctError(RuntimeError):
    pass


class StageSplitError(ValueError):
    pass


def lib():
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def check(status: int, what: str):
    if status == XCT_OK:
        return
    msg = lib().xct_last_error().decode(errors="replace")
    if status == XCT_ESTAGE:
        raise StageSplitError(f"{what}: {msg}")
    if status in (XCT_EINVAL, XCT_ENONFINITE):
        raise ValueError(f"{what}: {msg}")
    raise XctError(f"{what}: {msg} (status {status})")


# kernels launched per ABI call (for bench.py's gpu_launches count)
KERNELS_PER_CALL = {"xct_dot": 2, "xct_sum_f64": 1, "xct_spmm": 1, "xct_maxabs": 1,
                    "xct_chunk_maxabs": 1, "xct_normalize": 1, "xct_chunk_maxabs_chunked": 1,
                    "xct_normalize_chunked": 1, "xct_unchunk_f64": 1, "xct_chunk_from_f64": 1,
                    "xct_csr_spmm_f64": 1, "xct_siddon_count": 1, "xct_siddon_fill": 1,
                    "xct_csr_filter_cols": 1, "xct_csr_filter_map": 1, "xct_gather_rows": 1,
                    "xct_accumulate_rows": 1, "xct_scale_chunks": 2,
                    "xct_rows_to_chunked": 2, "xct_unchunk_rows_f64": 1,
                    "xct_siddon_project_f32": 1, "xct_fmtd_ranges": 1, "xct_fmtd_count": 1,
                    "xct_fmtd_fill": 1, "xct_csr_col_counts": 1,
                    "xct_ipc_alloc": (i32, [i64, C.POINTER(vp), vp]),
    "xct_ipc_open": (i32, [vp, C.POINTER(vp)]),
    "xct_ipc_close": (i32, [vp]),
    "xct_ipc_free": (i32, [vp]),
    "xct_gather_records": 1, "xct_accumulate_records": 1}
launch_count = [0]


def count_launches(name: str, n: int | None = None):
    launch_count[0] += KERNELS_PER_CALL.get(name, 0) if n is None else n


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)
    if name == "xct_axpy":      # second kernel when a sum of squares is requested
        count_launches(name, 2 if (args[8] is not None and args[13] is not None) else 1)
    else:
        count_launches(name)


def ptr(t) -> int | None:
    """Device/host address of a torch tensor or numpy array (None for None)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def n_threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


_STAGE_BYTES = 1 << 26
_stage = {}


def _staging(device):
    """Two reusable pinned host buffers (plus their copy-done events)."""
    import torch
    key = str(device)
    if key not in _stage:
        bufs = [torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        _stage[key] = (bufs, [b.numpy() for b in bufs],
                       [torch.cuda.Event() for _ in range(2)])
    return _stage[key]


def host_array(shape, dtype) -> np.ndarray:
    """A fresh host result array.  Large ones are anonymous mappings advised
    MADV_HUGEPAGE: filling a fresh 4 KiB-page array faults every page (17.7
    GB/s through the pinned staging on the B200 box), 2 MiB pages double it
    (34 GB/s, tools/d2h_hugepage_probe.py)."""
    import mmap
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    if n < (64 << 20) or not hasattr(mmap, "MADV_HUGEPAGE"):
        return np.empty(shape, dt)
    m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(m, dtype=dt).reshape(shape)


def to_host(t, out: np.ndarray | None = None) -> np.ndarray:
    """Device tensor -> numpy array (new, or the contiguous ``out`` of the
    same byte size), via double-buffered pinned staging (pageable ``.cpu()``
    runs at a few GB/s; the matrix builds move tens of GB this way)."""
    import torch
    t = t.contiguous()
    if out is None:
        out = np.empty(tuple(t.shape), dtype=torch.empty((), dtype=t.dtype).numpy().dtype)
    elif out.nbytes != t.numel() * t.element_size() or not out.flags.c_contiguous:
        raise ValueError("to_host: out does not match")
    n = t.numel() * t.element_size()
    if n == 0:
        return out
    if t.device.type != "cuda":
        out.reshape(-1).view(np.uint8)[:] = t.reshape(-1).view(torch.uint8).numpy()
        return out
    src = t.reshape(-1).view(torch.uint8)
    # host-side copies with torch (multi-threaded: the first touch of a
    # fresh result array is what a pageable .cpu() pays for, ~1 s per 2 GB)
    dst = torch.from_numpy(out.reshape(-1).view(np.uint8))
    bufs, views, evs = _staging(t.device)
    blocks = [(b, min(n, b + _STAGE_BYTES)) for b in range(0, n, _STAGE_BYTES)]
    for i, (b0, b1) in enumerate(blocks):
        bufs[i & 1][:b1 - b0].copy_(src[b0:b1], non_blocking=True)
        evs[i & 1].record()
        if i:
            p0, p1 = blocks[i - 1]
            evs[(i - 1) & 1].synchronize()
            dst[p0:p1].copy_(bufs[(i - 1) & 1][:p1 - p0])
    p0, p1 = blocks[-1]
    evs[(len(blocks) - 1) & 1].synchronize()
    dst[p0:p1].copy_(bufs[(len(blocks) - 1) & 1][:p1 - p0])
    return out


def to_device(a: np.ndarray, dst) -> None:
    """numpy array -> the contiguous device tensor ``dst`` (same byte size),
    via double-buffered pinned staging."""
    import torch
    a = np.ascontiguousarray(a)
    n = a.nbytes
    if n == 0:
        return
    if dst.numel() * dst.element_size() != n or not dst.is_contiguous():
        raise ValueError("to_device: size mismatch")
    src = a.reshape(-1).view(np.uint8)
    d = dst.reshape(-1).view(torch.uint8)
    if dst.device.type != "cuda":        # host-side (gloo) format copies
        d.copy_(torch.from_numpy(src))
        return
    bufs, views, evs = _staging(dst.device)
    for i, b0 in enumerate(range(0, n, _STAGE_BYTES)):
        b1 = min(n, b0 + _STAGE_BYTES)
        if i >= 2:
            evs[i & 1].synchronize()     # the copy that last used this buffer
        views[i & 1][:b1 - b0] = src[b0:b1]
        d[b0:b1].copy_(bufs[i & 1][:b1 - b0], non_blocking=True)
        evs[i & 1].record()
    for e in evs:
        e.synchronize()
