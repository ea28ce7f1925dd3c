"""Execution formats: staged, packed, device-resident operator sides.

Mirrors ``xct.matrixstore`` (src/matrixstore.py): precision policy
(storage/compute dtypes, element bytes), the power-of-two half rescale,
normalize/denormalize, StageSplitRequired -- and replaces build_staged/pack
(src/matrixstore.py:250-262, :417-562) with the B200 staged format built by
``xct_format_build`` and uploaded once to HBM.

A ``DeviceSide`` is one direction of the operator (projection A or back
projection A^T):

  * rows are grouped into CTA tiles: sinogram tiles (views x detectors) for
    A, voxel tiles (z x x) for A^T; tiles are launched in pseudo-Hilbert
    order;
  * each tile's input footprint is staged through shared memory in load
    groups: image bands perpendicular to the rays for A (so every row sees
    its entries in traversal order), view-angle ranges for A^T (so every
    voxel sees its rays in ascending ray id -- the reference order);
  * ``order="reference"`` keys A's groups by the reference's own stage ids
    (block_partitions x stage_capacity_bytes) instead, which reproduces the
    reference's per-row accumulation order bit for bit.

Record layout of a staged input element: f_dev slices x storage bytes, a
power of two in [16, 512] bytes; one lane owns 16 bytes of it.
"""

from __future__ import annotations

import ctypes as C
import functools
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .hilbert import pseudo_hilbert_cells

__all__ = ["PRECISIONS", "StageSplitRequired", "NormalizationState", "storage_dtype",
           "compute_dtype", "element_bytes", "half_rescale_exponent", "normalize",
           "denormalize", "DeviceSide", "build_device_side", "forward_plan", "adjoint_plan",
           "reference_plan", "row_block_plan", "f_dev_for", "DEFAULT_STAGE_CAPACITY",
           "SAFE_MAX"]

PRECISIONS = ("double", "single", "half", "mixed")
WARP_WIDTH = 32
DEFAULT_STAGE_CAPACITY = 96 * 1024      # src/matrixstore.py:44
SAFE_MAX = 60000.0                      # src/matrixstore.py:46
SMEM_BUDGET = 96 * 1024                 # per CTA: two resident CTAs per SM
SMEM_MAX = 224 * 1024                   # opt-in maximum per CTA on sm_100a
GROUPED_SMEM_BUDGET = 192 * 1024        # grouped rows: one CTA per SM

_STORE = {"double": np.float64, "single": np.float32, "half": np.float16, "mixed": np.float16}
_COMPUTE = {"double": np.float64, "single": np.float32, "half": np.float16, "mixed": np.float32}

StageSplitRequired = _lib.StageSplitError
INFO_FIELDS = [f for f, _ in _lib.FormatInfo._fields_]


def _check_precision(precision: str) -> None:
    if precision not in PRECISIONS:
        raise ValueError(f"unknown precision {precision!r}; expected one of {PRECISIONS}")


def storage_dtype(precision: str):
    _check_precision(precision)
    return _STORE[precision]


def compute_dtype(precision: str):
    _check_precision(precision)
    return _COMPUTE[precision]


def element_bytes(precision: str) -> int:
    return np.dtype(storage_dtype(precision)).itemsize


def f_dev_for(ffactor: int, precision: str) -> int:
    """Device slices per record: F rounded up so that the record is a power
    of two of at least 16 bytes (extra slices are zero and never written)."""
    eb = element_bytes(precision)
    rec = max(16, 1 << (int(ffactor) * eb - 1).bit_length())
    return rec // eb


def lanes_for(ffactor: int, precision: str, pieces_per_lane: int = 2) -> int:
    """Lanes sharing one row in K6: a record is f_dev*elem_bytes/16 pieces of
    16 bytes and every lane accumulates `pieces_per_lane` of them (measured
    on c2: one lane per row is fastest for FP16 and FP32 at F=16)."""
    pieces = f_dev_for(ffactor, precision) * element_bytes(precision) // 16
    return max(1, pieces // pieces_per_lane)


def half_rescale_exponent(values) -> int:
    """-floor(log2(median of the positive lengths)) (src/matrixstore.py:265-275).
    ``values`` may be a numpy array or a device tensor (median on the device,
    numpy's even-count convention: mean of the two middle values)."""
    if isinstance(values, np.ndarray):
        nz = values[values > 0]
        if len(nz) == 0:
            return 0
        return -int(math.floor(math.log2(float(np.median(nz)))))
    import torch
    nz = values[values > 0]
    n = int(nz.numel())
    if n == 0:
        return 0
    if n % 2:
        med = float(torch.kthvalue(nz, (n + 1) // 2).values)
    else:
        a = float(torch.kthvalue(nz, n // 2).values)
        b = float(torch.kthvalue(nz, n // 2 + 1).values)
        med = (a + b) / 2.0
    return -int(math.floor(math.log2(med)))


@dataclass
class NormalizationState:
    """Per-application scale (src/matrixstore.py:278-287)."""

    factor: float
    mode: str

    def __post_init__(self):
        if self.factor <= 0:
            raise ValueError("normalization factor must be positive")


def _peaks_to_factors(maxbits) -> list:
    peaks = maxbits.cpu().numpy().view(np.float64)
    if not np.all(np.isfinite(peaks)):
        raise ValueError("cannot normalize non-finite data")
    return [float(p) if p > 0 else 1.0 for p in peaks]


def normalize(vector, mode: str):
    """Max-abs scaling and cast to the storage dtype, on the device
    (src/matrixstore.py:290-305).  Returns (scaled, NormalizationState) with
    the same container type as the input (numpy in -> numpy out)."""
    import torch
    from .geometry import device
    _check_precision(mode)
    is_np = isinstance(vector, np.ndarray)
    dev = device()
    v = torch.as_tensor(np.asarray(vector) if is_np else vector, device=dev)
    if v.dtype not in (torch.float32, torch.float64):
        v = v.to(torch.float64)
    flat = v.reshape(-1, 1).contiguous()
    n = flat.shape[0]
    maxbits = torch.zeros(1, dtype=torch.int64, device=dev)
    st = _lib.stream_handle(dev)
    in64 = int(flat.dtype == torch.float64)
    _lib.call("xct_chunk_maxabs", _lib.ptr(flat), in64, n, 1, 1, 1, 1, _lib.ptr(maxbits), st)
    factor = _peaks_to_factors(maxbits)[0]
    fac = torch.tensor([factor], dtype=torch.float64, device=dev)
    sd = {"double": torch.float64, "single": torch.float32}.get(mode, torch.float16)
    out = torch.empty(n, dtype=sd, device=dev)
    # one chunk of one slice: record padding is irrelevant (f_dev = 1 here)
    _lib.call("xct_normalize", _lib.ptr(flat), in64, n, 1, 1, 1, 1, 1, _lib.ptr(fac),
              _lib.PREC_CODE[mode], _lib.ptr(out), st)
    out = out.reshape(v.shape)
    return (out.cpu().numpy() if is_np else out), NormalizationState(factor=factor, mode=mode)


def denormalize(vector, state: NormalizationState):
    """(src/matrixstore.py:308-316): f64 in double mode, f32 otherwise."""
    if isinstance(vector, np.ndarray):
        dt = np.float64 if state.mode == "double" else np.float32
        return vector.astype(dt) * dt(state.factor)
    import torch
    dt = torch.float64 if state.mode == "double" else torch.float32
    return vector.to(dt) * torch.tensor(state.factor, dtype=dt).item()


# ---------------------------------------------------------------------------
# CTA tiling / staging-key plans (host, integer, once per operator)
# ---------------------------------------------------------------------------

@dataclass
class Plan:
    """Rows per CTA tile plus the column keys that define the load groups."""

    cta_rows: np.ndarray          # int32 [n_cta, rows_per_cta], -1 = empty lane
    key_tables: np.ndarray        # int32 [n_tables, n_cols]
    cta_table: np.ndarray         # int32 [n_cta]
    rows_per_warp: int
    kind: str
    row_group: int = 1            # rows per unit (format_build row_group)


def _roundup(a, b):
    return -(-a // b) * b


def _unit_shape(kind: str, row_group: int):
    """(rows along the slow axis, along the fast axis) of one unit of
    `row_group` rows: views x detectors for A (adjacent views and detectors
    share most voxels: union/sum 0.80 for 2 views, 0.61 for 2x2), z x x for
    A^T (0.75 for a voxel pair, 0.50 for a 2x2 quad; measured, scale-free)."""
    if row_group == 1:
        return 1, 1
    if row_group == 2:
        return (2, 1) if kind == "forward" else (1, 2)
    if row_group == 4:
        return 2, 2
    raise ValueError("row_group must be 1, 2 or 4")


def forward_plan(num_angles: int, n: int, rows_per_warp: int, warps: int,
                 k0: int = 0, k1: int | None = None, row_group: int = 1) -> Plan:
    """Projection A (rows = rays k*N + c): CTA tiles of `ta` views x `td`
    detectors, one warp = rows_per_warp consecutive detectors of one view
    (row_group G > 1: one warp = G/gd views x rows_per_warp/G units of gd
    detectors, unit = the gv x gd rays one lane set owns).
    Load groups are image bands across the dominant ray direction: z bands
    for steep views, x bands (ascending for cos>0, descending for cos<0) for
    shallow ones, so a ray's entries stay in traversal order.
    [k0, k1) restricts the tiles to a range of views (k0 a multiple of the
    tile height); row ids stay global."""
    rw = rows_per_warp
    k1 = num_angles if k1 is None else k1
    if row_group > 1:
        gv, gd = _unit_shape("forward", row_group)
        upw = rw // row_group
        ud, uv = _grouped_forward_split(upw)          # units per warp: detectors x views
        td, ta = ud * gd, warps * uv * gv
        n_ta, n_td = -(-(k1 - k0) // ta), -(-n // td)
        cells = pseudo_hilbert_cells(n_td, n_ta)
        w, u, gi = np.meshgrid(np.arange(warps), np.arange(upw), np.arange(row_group),
                               indexing="ij")
        ai = ((w * uv + u // ud) * gv + gi // gd).reshape(-1)
        di = ((u % ud) * gd + gi % gd).reshape(-1)
    else:
        td = _forward_tile_width(n, rw, num_angles)
        rpc = max(td, (rw * warps) // td * td)
        ta = rpc // td
        n_ta, n_td = -(-(k1 - k0) // ta), -(-n // td)
        cells = pseudo_hilbert_cells(n_td, n_ta)           # (x = det tile, z = view tile)
        ai, di = np.divmod(np.arange(rpc), td)
        if _paired_setting() == "all" and td in (16, 32) and rw == 32 and ta % 2 == 0:
            # view-paired lanes: warp = 2 views x 16 detectors, lanes (2k, 2k+1)
            # = one detector in adjacent views (rays that share most voxels;
            # the paired half-warp schedule merges their LDS reads)
            w, ln = np.divmod(np.arange(rpc), 32)
            if td == 32:
                ai, di = 2 * (w // 2) + (ln & 1), 16 * (w % 2) + ln // 2
            else:
                ai, di = 2 * w + (ln & 1), ln // 2
    k = k0 + cells[:, 1:2] * ta + ai[None, :]
    c = cells[:, 0:1] * td + di[None, :]
    rows = np.where((k < k1) & (c < n), k * n + c, -1).astype(np.int32)
    return Plan(rows, _forward_key_tables(n), np.zeros(len(rows), np.int32), rw, "forward",
                row_group)


@functools.lru_cache(maxsize=4)
def _forward_key_tables(n: int) -> np.ndarray:
    """Band keys of every voxel column (z, x ascending, x descending); the
    same for every chunk of views, so built once (read-only)."""
    iz, ix = np.divmod(np.arange(n * n, dtype=np.int64), n)
    t = np.stack([iz, ix, n - 1 - ix]).astype(np.int32)
    t.flags.writeable = False
    return t


@functools.lru_cache(maxsize=4)
def _adjoint_key_tables(num_angles: int, n: int) -> np.ndarray:
    t = (np.arange(num_angles * n, dtype=np.int64) // n).astype(np.int32)[None, :]
    t.flags.writeable = False
    return t


def _forward_tile_width(n: int, rw: int, num_angles: int | None = None) -> int:
    """Detectors per forward CTA tile (one row per lane set): 16, i.e. tiles
    of 16 detectors x 32 views (a warp = 2 views x 16 detectors).  Measured
    at c5 (tools/spmm_probe.py): 32 x 16 952.6 ms, 16 x 32 937.3 ms (7.8 %
    fewer staged records per entry, 8 % fewer load groups), 8 x 64 1056 ms.
    XCT_FWD_TILE_DET overrides.  Fewer views than detectors (a tile's 32
    views then fan out by more than 32 x pi/N) keep 32 x 16: the wider
    footprint of 16 x 32 would exceed the device builder's 256 load groups
    per tile (measured at 2048^2 x 512 views)."""
    default = "16" if num_angles is None or num_angles >= n else "32"
    td = int(os.environ.get("XCT_FWD_TILE_DET", default))
    return min(_roundup(n, min(rw, td)), max(min(rw, td), td))


def _grouped_forward_split(upw: int) -> tuple:
    """A warp's units of grouped forward rows as (along detectors, along
    views): all along detectors unless XCT_FWD_GROUP_UD sets fewer."""
    ud = int(os.environ.get("XCT_FWD_GROUP_UD", "0")) or upw
    ud = max(1, min(upw, ud))
    while upw % ud:
        ud -= 1
    return ud, upw // ud


def forward_tile_height(n: int, rows_per_warp: int, warps: int, row_group: int = 1,
                        num_angles: int | None = None) -> int:
    if row_group > 1:
        ud, uv = _grouped_forward_split(rows_per_warp // row_group)
        return warps * uv * _unit_shape("forward", row_group)[0]
    rw = rows_per_warp
    td = _forward_tile_width(n, rw, num_angles)
    return max(td, (rw * warps) // td * td) // td


def assign_forward_regimes(plan: Plan, angles, n: int) -> Plan:
    """Pick the band key of every forward tile from its view angles: x
    bands (ascending for cos > 0, descending for cos < 0) when every view of
    the tile is shallow, z bands otherwise (z is non-decreasing along every
    ray since sin >= 0)."""
    ang = np.asarray(angles, dtype=np.float64)
    cs, sn = np.cos(ang), np.sin(ang)
    rows = plan.cta_rows
    valid = rows >= 0
    k = np.where(valid, rows // n, 0)
    shallow = np.abs(cs) > np.abs(sn)
    pos = shallow & (cs > 0)
    neg = shallow & (cs < 0)
    any_row = valid.any(axis=1)
    all_pos = np.all(np.where(valid, pos[k], True), axis=1) & any_row
    all_neg = np.all(np.where(valid, neg[k], True), axis=1) & any_row
    plan.cta_table = np.where(all_pos, 1, np.where(all_neg, 2, 0)).astype(np.int32)
    return plan


def adjoint_plan(num_angles: int, n: int, rows_per_warp: int, warps: int,
                 z0: int = 0, z1: int | None = None, row_group: int = 1) -> Plan:
    """Back projection A^T (rows = voxels iz*N + ix): CTA tiles of tz x tx
    voxels, a warp = rows_per_warp consecutive voxels of one image row
    (row_group G > 1: a warp = gz image rows x rows_per_warp/G units of gx
    voxels, unit = the gz x gx voxels one lane set owns).
    Load groups are ranges of view angles (key = ray // N).  [z0, z1)
    restricts the tiles to a band of image rows (z0 a multiple of tz)."""
    rw = rows_per_warp
    z1 = n if z1 is None else z1
    if row_group > 1:
        gz, gx = _unit_shape("adjoint", row_group)
        upw = rw // row_group
        tx, tz = upw * gx, warps * gz
        n_tz, n_tx = -(-(z1 - z0) // tz), -(-n // tx)
        cells = pseudo_hilbert_cells(n_tx, n_tz)
        w, u, gi = np.meshgrid(np.arange(warps), np.arange(upw), np.arange(row_group),
                               indexing="ij")
        zi = (w * gz + gi // gx).reshape(-1)
        xi = (u * gx + gi % gx).reshape(-1)
    else:
        tx = _adjoint_tile_width(n, rw)
        rpc = max(tx, (rw * warps) // tx * tx)
        tz = rpc // tx
        n_tz, n_tx = -(-(z1 - z0) // tz), -(-n // tx)
        cells = pseudo_hilbert_cells(n_tx, n_tz)
        zi, xi = np.divmod(np.arange(rpc), tx)
    z = z0 + cells[:, 1:2] * tz + zi[None, :]
    x = cells[:, 0:1] * tx + xi[None, :]
    rows = np.where((z < z1) & (x < n), z * n + x, -1).astype(np.int32)
    return Plan(rows, _adjoint_key_tables(num_angles, n), np.zeros(len(rows), np.int32), rw,
                "adjoint", row_group)


def _adjoint_tile_width(n: int, rw: int) -> int:
    """Voxels along x per back-projection CTA tile (one row per lane set):
    16, i.e. tiles of 16 x 32 voxels (a warp = 2 image rows x 16 voxels).
    Measured at c5 (tools/spmm_probe.py): 32 x 16 825 ms, 16 x 32 811 ms
    (same footprint, padding 1.095 -> 1.088), 64 x 8 946 ms.
    XCT_ADJ_TILE_X overrides."""
    tx = int(os.environ.get("XCT_ADJ_TILE_X", "16"))
    return min(_roundup(n, min(rw, tx)), max(min(rw, tx), tx))


def adjoint_tile_height(n: int, rows_per_warp: int, warps: int, row_group: int = 1) -> int:
    if row_group > 1:
        return warps * _unit_shape("adjoint", row_group)[0]
    rw = rows_per_warp
    tx = _adjoint_tile_width(n, rw)
    return max(tx, (rw * warps) // tx * tx) // tx


def restrict_plan(plan: Plan, row_ids: np.ndarray, col_ids: np.ndarray) -> Plan:
    """A plan over a block of the operator (rows = global `row_ids`, local
    columns = global `col_ids`): the global tiles restricted to the block's
    rows (renumbered to local positions, empty tiles dropped) and the key
    tables re-indexed by the local columns."""
    pos = np.full(int(max(plan.cta_rows.max(), row_ids.max() if len(row_ids) else 0)) + 1, -1,
                  np.int64)
    pos[row_ids] = np.arange(len(row_ids))
    rows = np.where(plan.cta_rows >= 0, pos[np.maximum(plan.cta_rows, 0)], -1)
    keep = (rows >= 0).any(axis=1)
    return Plan(rows[keep].astype(np.int32), plan.key_tables[:, col_ids],
                plan.cta_table[keep], plan.rows_per_warp, plan.kind, plan.row_group)


def row_block_plan(n_rows: int, n_cols: int, rows_per_warp: int, warps: int,
                   keys: np.ndarray | None = None, row_group: int = 1) -> Plan:
    """Consecutive rows per CTA, one key table (default: one key per column
    range of 1 -- i.e. groups are column ranges)."""
    rpc = rows_per_warp * warps
    n_cta = max(1, -(-n_rows // rpc))
    r = np.arange(n_cta * rpc)
    rows = np.where(r < n_rows, r, -1).astype(np.int32).reshape(n_cta, rpc)
    if keys is None:
        keys = np.arange(n_cols, dtype=np.int32)
    return Plan(rows, np.asarray(keys, np.int32)[None, :], np.zeros(n_cta, np.int32),
                rows_per_warp, "rows", row_group)


def reference_plan(indptr: np.ndarray, indices: np.ndarray, n_rows: int, n_cols: int,
                   block_partitions: int, stage_capacity_bytes, ffactor: int, precision: str,
                   rows_per_warp: int, warps: int) -> Plan:
    """Keys = the reference's stage ids: rows split into `block_partitions`
    contiguous chunks, each chunk's sorted footprint cut every
    cap // (elem_bytes * F) columns (src/matrixstore.py:434-485).  CTA tiles
    never straddle a chunk, so each row's accumulation order is exactly the
    reference's (stage, traversal) order."""
    eb = element_bytes(precision)
    parts = min(block_partitions, max(1, n_rows))
    base, rem = divmod(n_rows, parts)
    bounds = np.concatenate(([0], np.cumsum([base + (i < rem) for i in range(parts)])))
    tables = np.zeros((parts, n_cols), np.int32)
    rpc = rows_per_warp * warps
    rows_list, tab_list = [], []
    for p in range(parts):
        lo, hi = indptr[bounds[p]], indptr[bounds[p + 1]]
        fp = np.unique(indices[lo:hi])
        if stage_capacity_bytes is None:
            cap = max(1, len(fp))
        else:
            cap = stage_capacity_bytes // (eb * ffactor)
            if cap < 1:
                raise ValueError(
                    f"stage capacity {stage_capacity_bytes} B cannot hold one element at "
                    f"{precision} precision with fusing factor {ffactor}")
        cap = min(cap, 65536)
        tables[p, fp] = (np.arange(len(fp)) // cap).astype(np.int32)
        r0, r1 = bounds[p], bounds[p + 1]
        for s in range(r0, r1, rpc):
            blk = np.full(rpc, -1, np.int32)
            e = min(r1, s + rpc)
            blk[:e - s] = np.arange(s, e)
            rows_list.append(blk)
            tab_list.append(p)
    if not rows_list:
        rows_list = [np.full(rpc, -1, np.int32)]
        tab_list = [0]
    return Plan(np.stack(rows_list), tables, np.asarray(tab_list, np.int32), rows_per_warp,
                "reference")


# ---------------------------------------------------------------------------
# device-resident side
# ---------------------------------------------------------------------------

@dataclass
class DeviceSide:
    """One staged operator direction in HBM (kernel K6 input)."""

    precision: str
    ffactor: int
    f_dev: int
    n_in: int
    n_out: int
    value_scale_exp: int
    info: _lib.FormatInfo
    tensors: dict = field(repr=False)
    staged: _lib.Staged = field(repr=False, default=None)
    smem_bytes: int = 0
    plan_kind: str = ""
    contract: bool = False       # single: FFMA instead of multiply-then-add
    chunk_group: int = 1         # F-chunks of a tile launched adjacently

    @property
    def nnz(self) -> int:
        return int(self.info.nnz)

    @property
    def padded_entries(self) -> int:
        return int(self.info.n_padded)

    @property
    def entry_bytes(self) -> int:
        return 2 + int(self.info.value_bytes)

    def hbm_bytes(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in self.tensors.values())


@dataclass
class HostFormat:
    """Exported K5 format on the host (exact-size arrays) plus its rows."""

    arrays: dict
    info: dict
    cta_rows: np.ndarray
    plan_kind: str


def build_format(indptr: np.ndarray, indices32: np.ndarray, values: np.ndarray,
                 n_rows: int, n_cols: int, plan: Plan, precision: str, ffactor: int,
                 value_scale_exp: int, smem_budget: int = SMEM_BUDGET,
                 schedule: bool = False) -> HostFormat:
    """Run the K5 host builder (libxct_b200) and export its arrays."""
    _check_precision(precision)
    f_dev = f_dev_for(ffactor, precision)
    rec = f_dev * element_bytes(precision)
    # the kernel double-buffers the stage: two groups of `capacity` records
    # K6 addresses a staged record by a 16-bit byte offset (slot * 16)
    capacity = min(65536 // 16, max(1, smem_budget // (2 * rec)))
    rows = np.ascontiguousarray(plan.cta_rows, np.int32)
    keys = np.ascontiguousarray(plan.key_tables, np.int32)
    ctab = np.ascontiguousarray(plan.cta_table, np.int32)
    ip = np.ascontiguousarray(indptr, np.int64)
    ix = np.ascontiguousarray(indices32, np.int32)
    vals = np.ascontiguousarray(values, np.float64)
    handle = C.c_void_p()
    L = _lib.lib()
    lp = (rec // 16).bit_length() - 1
    G = int(plan.row_group)
    lg = (32 // (plan.rows_per_warp // G)).bit_length() - 1
    st = L.xct_format_build(n_rows, n_cols, ip.ctypes.data, ix.ctypes.data if len(ix) else None,
                            vals.ctypes.data if len(vals) else None,
                            rows.shape[0], rows.shape[1], plan.rows_per_warp,
                            rows.ctypes.data, keys.ctypes.data, ctab.ctypes.data, capacity,
                            _lib.PREC_CODE[precision], int(value_scale_exp),
                            lp if schedule else -1, lg if schedule else -1, G,
                            _lib.n_threads(), C.byref(handle))
    _lib.check(st, "xct_format_build")
    try:
        info = _lib.FormatInfo()
        _lib.check(L.xct_format_get_info(handle, C.byref(info)), "xct_format_get_info")
        warps = int(info.warps_per_cta)
        sizes = dict(cta_group_ptr=info.n_cta + 1, group_map_ptr=info.n_groups + 1,
                     group_map=info.n_slots, slab_off=info.n_groups * warps,
                     slab_width=info.n_groups * warps, slots=info.n_padded,
                     values=info.n_padded * max(1, int(info.row_group)))
        dts = dict(cta_group_ptr=np.int32, group_map_ptr=np.int64, group_map=np.int32,
                   slab_off=np.int64, slab_width=np.int32, slots=np.uint16,
                   values=storage_dtype(precision))
        h = {k: np.empty(max(int(n), 1), dts[k]) for k, n in sizes.items()}
        _lib.check(L.xct_format_export(handle, *[h[k].ctypes.data for k in
                                                 ("cta_group_ptr", "group_map_ptr", "group_map",
                                                  "slab_off", "slab_width", "slots", "values")]),
                   "xct_format_export")
    finally:
        L.xct_format_free(handle)
    h = {k: v[:int(sizes[k])] for k, v in h.items()}
    return HostFormat(h, {f: getattr(info, f) for f in INFO_FIELDS}, rows.reshape(-1),
                      plan.kind)


def concat_formats(parts: list) -> HostFormat:
    """Concatenate formats of disjoint CTA-tile sets built separately (e.g.
    streamed over angle or voxel chunks): offsets are rebased."""
    if len(parts) == 1:
        return parts[0]
    i0 = parts[0].info
    out = {k: [] for k in parts[0].arrays}
    rows = []
    g_off = s_off = e_off = 0
    for hf in parts:
        a, inf = hf.arrays, hf.info
        for k in ("rows_per_cta", "rows_per_warp", "warps_per_cta", "value_bytes", "row_group"):
            if inf[k] != i0[k]:
                raise ValueError(f"cannot concatenate formats with different {k}")
        out["cta_group_ptr"].append(a["cta_group_ptr"][:-1] + g_off)
        out["group_map_ptr"].append(a["group_map_ptr"][:-1] + s_off)
        out["group_map"].append(a["group_map"])
        out["slab_off"].append(a["slab_off"] + e_off)
        out["slab_width"].append(a["slab_width"])
        out["slots"].append(a["slots"])
        out["values"].append(a["values"])
        rows.append(hf.cta_rows)
        g_off += int(inf["n_groups"])
        s_off += int(inf["n_slots"])
        e_off += int(inf["n_padded"])
    out["cta_group_ptr"].append(np.array([g_off], np.int32))
    out["group_map_ptr"].append(np.array([s_off], np.int64))
    arrays = {k: np.concatenate(v) for k, v in out.items()}
    info = dict(i0)
    for k in ("n_cta", "n_groups", "n_slots", "n_padded", "nnz", "underflow_count"):
        info[k] = sum(int(hf.info[k]) for hf in parts)
    info["max_group_slots"] = max(int(hf.info["max_group_slots"]) for hf in parts)
    info["max_rel_quant_error"] = max(float(hf.info["max_rel_quant_error"]) for hf in parts)
    return HostFormat(arrays, info, np.concatenate(rows), parts[0].plan_kind)


def upload_format(hf, precision: str, ffactor: int, n_in: int, n_out: int,
                  value_scale_exp: int, dev=None) -> "DeviceSide":
    """Encode the entries for K6 and move the format (a HostFormat or a list
    of parts over disjoint CTA tiles) to HBM.  Parts are rebased and copied
    straight into the final device arrays, in bounded host blocks, so no
    whole-operator host copy is ever made."""
    import torch
    from .geometry import device
    dev = dev or device()
    parts = hf if isinstance(hf, list) else [hf]
    i0 = parts[0].info
    for p in parts:
        for k in ("rows_per_cta", "rows_per_warp", "warps_per_cta", "value_bytes", "row_group"):
            if p.info[k] != i0[k]:
                raise ValueError(f"cannot combine formats with different {k}")
    tot = {k: sum(int(p.info[k]) for p in parts)
           for k in ("n_cta", "n_groups", "n_slots", "n_padded", "nnz", "underflow_count")}
    info = _lib.FormatInfo()
    for f, v in i0.items():
        setattr(info, f, v)
    for k, v in tot.items():
        setattr(info, k, v)
    info.max_group_slots = max(int(p.info["max_group_slots"]) for p in parts)
    info.max_rel_quant_error = max(float(p.info["max_rel_quant_error"]) for p in parts)
    f_dev = f_dev_for(ffactor, precision)
    # K6 addresses a staged record by its byte offset inside a plane
    plane_slots = -(-int(info.max_group_slots) // 8) * 8
    if plane_slots * 16 > 65536:
        raise StageSplitRequired("load group too large for 16-bit plane offsets")
    G = max(1, int(info.row_group))
    packed = precision in ("half", "mixed") and G == 1
    warps = int(info.warps_per_cta)
    pad = 1024          # the kernel's load ring reads up to 4 steps past a slab
    T = {}

    def alloc(name, n, dtype):
        T[name] = torch.zeros(max(int(n), 1), dtype=dtype, device=dev)
    alloc("cta_group_ptr", tot["n_cta"] + 1, torch.int32)
    alloc("group_map_ptr", tot["n_groups"] + 1, torch.int64)
    alloc("group_map", tot["n_slots"], torch.int32)
    alloc("slab_off", tot["n_groups"] * warps, torch.int64)
    alloc("slab_width", tot["n_groups"] * warps, torch.int32)
    alloc("cta_rows", tot["n_cta"] * int(info.rows_per_cta), torch.int32)
    if packed:
        alloc("values", tot["n_padded"] + pad, torch.int32)
        alloc("slots", 1, torch.int16)
    elif G > 1:         # grouped rows: u16 offsets + G values per position
        alloc("values", (tot["n_padded"] + pad) * G,
              torch.int16 if precision == "mixed" else torch.float32)
        alloc("slots", tot["n_padded"] + pad, torch.int16)
    else:
        alloc("values", tot["n_padded"] + pad,
              torch.float64 if precision == "double" else torch.float32)
        alloc("slots", tot["n_padded"] + pad, torch.int16)

    def put(name, at, arr):
        if len(arr):
            _lib.to_device(arr, T[name][at:at + len(arr)])

    c_off = g_off = s_off = e_off = r_off = 0
    block = 1 << 25
    for p in parts:
        a, inf = p.arrays, p.info
        put("cta_group_ptr", c_off, a["cta_group_ptr"][:-1] + g_off)
        put("group_map_ptr", g_off, a["group_map_ptr"][:-1] + s_off)
        put("group_map", s_off, a["group_map"])
        put("slab_off", g_off * warps, a["slab_off"] + e_off)
        put("slab_width", g_off * warps, a["slab_width"])
        put("cta_rows", r_off, p.cta_rows)
        n = int(inf["n_padded"])
        for b0 in range(0, n, block):
            # records are packed on the device: offset = slot*16, and for
            # half/mixed word = offset<<16 | fp16 bits
            b1 = min(n, b0 + block)
            ds = torch.empty(b1 - b0, dtype=torch.int16, device=dev)
            _lib.to_device(a["slots"][b0:b1].view(np.int16), ds)
            off = (ds.to(torch.int64) & 0xFFFF) << 4
            if G > 1:
                T["slots"][e_off + b0:e_off + b1].copy_(off.view(torch.int16)[0::4])
                vv = a["values"][b0 * G:b1 * G]
                put("values", (e_off + b0) * G, vv.view(np.int16) if precision == "mixed" else vv)
            elif packed:
                dv = torch.empty(b1 - b0, dtype=torch.int16, device=dev)
                _lib.to_device(a["values"][b0:b1].view(np.int16), dv)
                word = (off << 16) | (dv.to(torch.int64) & 0xFFFF)
                T["values"][e_off + b0:e_off + b1].copy_(word.view(torch.int32)[0::2])
            else:
                T["slots"][e_off + b0:e_off + b1].copy_(off.view(torch.int16)[0::4])
                put("values", e_off + b0, a["values"][b0:b1])
        c_off += int(inf["n_cta"])
        g_off += int(inf["n_groups"])
        s_off += int(inf["n_slots"])
        e_off += n
        r_off += len(p.cta_rows)
    T["cta_group_ptr"][tot["n_cta"]] = g_off
    T["group_map_ptr"][tot["n_groups"]] = s_off
    side = DeviceSide(precision, ffactor, f_dev, n_in, n_out, value_scale_exp, info, T,
                      plan_kind=parts[0].plan_kind)
    return attach(side)


# ---------------------------------------------------------------------------
# K5 on the device (csrc/format_device.cu): same arrays as build_format +
# upload_format for the band / view-key plans with one row per lane set
# ---------------------------------------------------------------------------

PAD_ENTRIES = 1024      # the kernel's load ring reads up to 4 steps past a slab


class DeviceBuildUnsupported(Exception):
    """The device builder declined (limits or row order): use the host one."""


def device_build_supported(plan: Plan, precision: str) -> bool:
    return plan.kind in ("forward", "adjoint") and int(plan.row_group) == 1 and \
        os.environ.get("XCT_HOST_BUILD") != "1"


def _sched_rq(plan: Plan, precision: str, ffactor: int, schedule: bool) -> int:
    """Rows per quarter-warp of the bank model (format_build.cpp BankModel)."""
    if not schedule:
        return 0
    lg = (32 // plan.rows_per_warp).bit_length() - 1
    return (8 >> lg) if lg <= 3 else 1


def _paired_setting() -> str:
    """XCT_FMTD_PAIRED: "adjoint" (default: the paired half-warp schedule
    for A^T), "all" (also A, with view-paired forward lanes), "0" (off)."""
    return os.environ.get("XCT_FMTD_PAIRED", "adjoint")


def _sched_mode(exact: bool, kind: str = "forward") -> int:
    """0: the host's schedule exactly (raises where it cannot run); 1
    (default): the host's schedule, first fit where a slab exceeds its
    limits (image-corner tiles); 2: first fit everywhere (fastest build,
    ~3% slower K6 at c5 from more bank conflicts, r02 measurement); 3/4:
    the paired half-warp schedule (one LDS wavefront per half-warp where
    row pairs share records; format_device.cu paired_half), 4 with only
    the entries the merged steps cannot hold on the per-quarter steps (the
    default for A^T; 3 fills those steps first)."""
    if exact or os.environ.get("XCT_FMTD_EXACT") == "1":
        return 0
    if os.environ.get("XCT_FMTD_FAST") == "1":
        return 2
    paired = _paired_setting()
    if paired == "all" or (paired == "adjoint" and kind == "adjoint"):
        mode = 3 if os.environ.get("XCT_FMTD_PAIRED_FILL") == "1" else 4
        extra = int(os.environ.get("XCT_FMTD_PAIRED_EXTRA", "20"))  # % of F, slack steps
        # first-fit colourings (no alternating paths): 27 % less fill time;
        # for A also fewer modelled wavefronts (used there), for A^T +2.6 %
        # of them (c5: 1,793.5 -> 1,802.1 ms/iter for assembly 31.6 -> 29.4 s,
        # and c1's native-order deviation from the reference 1.4e-3 ->
        # 2.5e-3, closer to its bound): A^T keeps the alternating-path
        # colourer unless XCT_FMTD_PAIRED_GREEDY=1
        greedy = 1 if (kind == "forward" or
                       os.environ.get("XCT_FMTD_PAIRED_GREEDY") == "1") else 0
        return mode | (min(max(extra, 0), 255) << 8) | (greedy << 16)
    return 1


@dataclass
class DevicePart:
    """One part (a chunk of views / a band of voxels) of a device-built side."""

    tensors: dict
    info: dict
    cta_rows: np.ndarray
    plan_kind: str


def build_format_device(d_indptr, d_indices, d_values, n_rows: int, n_cols: int, plan: Plan,
                        precision: str, ffactor: int, value_scale_exp: int, smem_budget: int,
                        schedule: bool, base_b: int, n_keys: int, dev, pad: bool = True,
                        exact: bool = False) -> DevicePart:
    """Device K5 of one part: ``d_*`` is the part's device CSR (row ids as in
    ``plan.cta_rows``, global column ids); ``base_b``/``n_keys`` define the
    key/coordinate of a column (grid_n, grid_n for A; detectors, views for
    A^T).  ``exact`` runs the host's bank schedule step for step (byte-
    identical to build_format; one thread per quarter-warp, slow at scale);
    the default first-fit schedule places the same entries in the same
    slabs on other steps.  Raises DeviceBuildUnsupported when the host
    builder must do it."""
    import torch
    if not device_build_supported(plan, precision):
        raise DeviceBuildUnsupported("plan kind or row group")
    f_dev = f_dev_for(ffactor, precision)
    rec = f_dev * element_bytes(precision)
    capacity = min(65536 // 16, max(1, smem_budget // (2 * rec)))
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    rows = np.ascontiguousarray(plan.cta_rows, np.int32)
    n_cta, rpc = rows.shape
    rpw = int(plan.rows_per_warp)
    warps = rpc // rpw
    d_rows = torch.from_numpy(rows.reshape(-1)).to(dev)
    modes = np.ascontiguousarray(plan.cta_table, np.int32) if plan.kind == "forward" \
        else np.zeros(n_cta, np.int32)
    d_modes = torch.from_numpy(modes).to(dev)
    part = _lib.FmtdPart(d_indptr.data_ptr(), d_indices.data_ptr(), d_values.data_ptr(),
                         int(n_rows), d_rows.data_ptr(), d_modes.data_ptr(), int(n_cta), int(rpc),
                         rpw, int(base_b), int(n_keys), int(capacity),
                         _sched_rq(plan, precision, ffactor, schedule),
                         _sched_mode(exact, plan.kind))
    i32, i64 = torch.int32, torch.int64
    flag = torch.zeros(1, dtype=i32, device=dev)
    lo = torch.empty(max(n_cta * n_keys, 1), dtype=i32, device=dev)
    hi = torch.empty_like(lo)
    span = torch.zeros(max(n_cta, 1), dtype=i64, device=dev)
    _lib.check(L.xct_fmtd_ranges(C.byref(part), lo.data_ptr(), hi.data_ptr(), span.data_ptr(),
                                 flag.data_ptr(), st), "xct_fmtd_ranges")
    bm_words = int(span.max().item()) // 32 + 2 if n_cta else 1
    counts = torch.zeros((max(n_cta, 1), 4), dtype=i64, device=dev)
    widths = torch.zeros(max(n_cta, 1) * 256 * warps, dtype=i32, device=dev)
    stc = L.xct_fmtd_count(C.byref(part), lo.data_ptr(), hi.data_ptr(), bm_words,
                           counts.data_ptr(), widths.data_ptr(), flag.data_ptr(), st)
    if stc == _lib.XCT_ESTAGE:
        raise DeviceBuildUnsupported("tile footprint exceeds shared memory")
    _lib.check(stc, "xct_fmtd_count")
    fl = int(flag.item())
    if fl:
        raise DeviceBuildUnsupported(f"count flags {fl}")
    cnt = counts.cpu().numpy()[:n_cta]
    ng, ns, mgs, npad = (cnt[:, i] for i in range(4))
    base = np.zeros((max(n_cta, 1), 3), np.int64)
    base[1:n_cta, 0] = np.cumsum(ng)[:-1]
    base[1:n_cta, 1] = np.cumsum(ns)[:-1]
    base[1:n_cta, 2] = np.cumsum(npad)[:-1]
    n_groups, n_slots, n_padded = int(ng.sum()), int(ns.sum()), int(npad.sum())
    T = {}
    T["cta_group_ptr"] = torch.from_numpy(
        np.concatenate(([0], np.cumsum(ng))).astype(np.int32)).to(dev)
    T["group_map_ptr"] = torch.zeros(n_groups + 1, dtype=i64, device=dev)
    T["group_map"] = torch.zeros(max(n_slots, 1), dtype=i32, device=dev)
    T["slab_off"] = torch.zeros(max(n_groups * warps, 1), dtype=i64, device=dev)
    T["slab_width"] = torch.zeros(max(n_groups * warps, 1), dtype=i32, device=dev)
    T["cta_rows"] = d_rows
    extra = PAD_ENTRIES if pad else 0
    packed = precision in ("half", "mixed")
    if packed:
        T["values"] = torch.zeros(n_padded + extra, dtype=i32, device=dev)
        T["slots"] = torch.zeros(1, dtype=torch.int16, device=dev)
    else:
        T["values"] = torch.zeros(n_padded + extra, dtype=torch.float64 if precision == "double"
                                  else torch.float32, device=dev)
        T["slots"] = torch.zeros(n_padded + extra, dtype=torch.int16, device=dev)
    # per call (the caching allocator hands the block back to later builds
    # and, after assembly, to the solver's vectors); the fill runs
    # min(n_cta, 2 x 148) CTAs, so small parts need a fraction of it
    full = int(L.xct_fmtd_scratch_bytes())
    ctas = min(int(n_cta), 2 * 148)
    scratch = torch.empty(max(1, full * ctas // (2 * 148)), dtype=torch.uint8, device=dev)
    qs = torch.zeros(7, dtype=i64, device=dev)
    d_base = torch.from_numpy(base).to(dev)
    _lib.check(L.xct_fmtd_fill(C.byref(part), lo.data_ptr(), hi.data_ptr(), bm_words,
                               widths.data_ptr(), d_base.data_ptr(), _lib.PREC_CODE[precision],
                               int(value_scale_exp), T["group_map"].data_ptr(),
                               T["group_map_ptr"].data_ptr(), T["slab_off"].data_ptr(),
                               T["slab_width"].data_ptr(),
                               None if packed else T["slots"].data_ptr(), T["values"].data_ptr(),
                               scratch.data_ptr(), scratch.numel(), flag.data_ptr(), qs.data_ptr(),
                               st), "xct_fmtd_fill")
    fl = int(flag.item())
    if fl:
        raise DeviceBuildUnsupported(f"fill flags {fl}, widest slab {int(widths.max())} steps")
    q = qs.cpu().numpy()
    nnz = int((d_indptr[n_rows] - d_indptr[0]).item())
    info = dict(n_cta=int(n_cta), rows_per_cta=int(rpc), rows_per_warp=rpw,
                warps_per_cta=int(warps), n_groups=n_groups, n_slots=n_slots, n_padded=n_padded,
                nnz=nnz, max_group_slots=int(mgs.max()) if n_cta else 0,
                value_bytes=element_bytes(precision),
                max_rel_quant_error=float(q[:1].view(np.float64)[0]),
                underflow_count=int(q[1]), row_group=1)
    if q[3]:
        info["paired_merged_steps"], info["paired_half_steps"] = int(q[2]), int(q[3])
        info["paired_conflicts"] = {"quarter_steps": int(q[4]), "merged_steps": int(q[5])}
        info["paired_fallback_halves"] = int(q[6])
    return DevicePart(T, info, rows.reshape(-1), plan.kind)


def host_part(hf: "HostFormat", precision: str, ffactor: int, n_in: int, n_out: int,
              value_scale_exp: int, dev) -> DevicePart:
    """A host-built part (e.g. grouped rows, which the device builder does
    not make) uploaded and wrapped as a DevicePart for combine_device_parts."""
    side = upload_format(hf, precision, ffactor, n_in, n_out, value_scale_exp, dev)
    info = {f: getattr(side.info, f) for f in INFO_FIELDS}
    return DevicePart(side.tensors, info, hf.cta_rows, hf.plan_kind)


def combine_device_parts(parts: list, precision: str, ffactor: int, n_in: int, n_out: int,
                         value_scale_exp: int, dev) -> "DeviceSide":
    """Concatenate device-built parts over disjoint CTA tiles (offsets
    rebased, as upload_format does for host parts); each part's tensors are
    released as soon as they are copied."""
    import torch
    f_dev = f_dev_for(ffactor, precision)
    if len(parts) == 1:
        P = parts[0]
        T = P.tensors
        parts.clear()
    else:
        tot = {k: sum(int(p.info[k]) for p in parts)
               for k in ("n_cta", "n_groups", "n_slots", "n_padded")}
        warps = int(parts[0].info["warps_per_cta"])
        rpc = int(parts[0].info["rows_per_cta"])
        packed = precision in ("half", "mixed")
        T = {"cta_group_ptr": torch.empty(tot["n_cta"] + 1, dtype=torch.int32, device=dev),
             "group_map_ptr": torch.empty(tot["n_groups"] + 1, dtype=torch.int64, device=dev),
             "group_map": torch.empty(max(tot["n_slots"], 1), dtype=torch.int32, device=dev),
             "slab_off": torch.empty(max(tot["n_groups"] * warps, 1), dtype=torch.int64,
                                     device=dev),
             "slab_width": torch.empty(max(tot["n_groups"] * warps, 1), dtype=torch.int32,
                                       device=dev),
             "cta_rows": torch.empty(tot["n_cta"] * rpc, dtype=torch.int32, device=dev)}
        vt = parts[0].tensors["values"].dtype
        G = max(1, int(parts[0].info.get("row_group", 1)))
        packed = packed and G == 1
        T["values"] = torch.zeros((tot["n_padded"] + PAD_ENTRIES) * G, dtype=vt, device=dev)
        T["slots"] = (torch.zeros(1, dtype=torch.int16, device=dev) if packed else
                      torch.zeros(tot["n_padded"] + PAD_ENTRIES, dtype=torch.int16, device=dev))
        c_off = g_off = s_off = e_off = 0
        infos = [p.info for p in parts]
        for P in parts:
            A, inf = P.tensors, P.info
            nc, ng = int(inf["n_cta"]), int(inf["n_groups"])
            ns, ne = int(inf["n_slots"]), int(inf["n_padded"])
            T["cta_group_ptr"][c_off:c_off + nc] = A["cta_group_ptr"][:nc] + g_off
            T["group_map_ptr"][g_off:g_off + ng] = A["group_map_ptr"][:ng] + s_off
            T["group_map"][s_off:s_off + ns] = A["group_map"][:ns]
            T["slab_off"][g_off * warps:(g_off + ng) * warps] = A["slab_off"][:ng * warps] + e_off
            T["slab_width"][g_off * warps:(g_off + ng) * warps] = A["slab_width"][:ng * warps]
            T["cta_rows"][c_off * rpc:(c_off + nc) * rpc] = A["cta_rows"][:nc * rpc]
            T["values"][e_off * G:(e_off + ne) * G] = A["values"][:ne * G]
            if not packed:
                T["slots"][e_off:e_off + ne] = A["slots"][:ne]
            P.tensors = None               # release this part's device arrays
            c_off, g_off, s_off, e_off = c_off + nc, g_off + ng, s_off + ns, e_off + ne
        T["cta_group_ptr"][c_off] = g_off
        T["group_map_ptr"][g_off] = s_off
        P = parts[0]
        P.info = dict(infos[0])
        for k in ("n_cta", "n_groups", "n_slots", "n_padded", "nnz", "underflow_count"):
            P.info[k] = sum(int(i[k]) for i in infos)
        P.info["max_group_slots"] = max(int(i["max_group_slots"]) for i in infos)
        P.info["max_rel_quant_error"] = max(float(i["max_rel_quant_error"]) for i in infos)
        parts.clear()
    info = _lib.FormatInfo()
    for f, v in P.info.items():
        setattr(info, f, v)
    plane_slots = -(-int(info.max_group_slots) // 8) * 8
    if plane_slots * 16 > 65536:
        raise StageSplitRequired("load group too large for 16-bit plane offsets")
    side = DeviceSide(precision, ffactor, f_dev, n_in, n_out, value_scale_exp, info, T,
                      plan_kind=P.plan_kind)
    return attach(side)


def build_device_side(indptr: np.ndarray, indices32: np.ndarray, values: np.ndarray,
                      n_rows: int, n_cols: int, plan: Plan, precision: str, ffactor: int,
                      value_scale_exp: int, smem_budget: int = SMEM_BUDGET,
                      dev=None, schedule: bool = False) -> "DeviceSide":
    """Build the staged format on the host (libxct_b200 K5) and upload it."""
    hf = build_format(indptr, indices32, values, n_rows, n_cols, plan, precision, ffactor,
                      value_scale_exp, smem_budget, schedule)
    return upload_format(hf, precision, ffactor, n_cols, n_rows, value_scale_exp, dev)


def attach(side: DeviceSide) -> DeviceSide:
    """(Re)bind the kernel descriptor of a side to its device tensors."""
    info, t = side.info, side.tensors
    s = _lib.Staged()
    s.n_cta, s.rows_per_cta = info.n_cta, info.rows_per_cta
    s.warps_per_cta, s.rows_per_warp = info.warps_per_cta, info.rows_per_warp
    s.n_groups, s.max_group_slots = info.n_groups, info.max_group_slots
    s.d_cta_rows = t["cta_rows"].data_ptr()
    s.d_cta_group_ptr = t["cta_group_ptr"].data_ptr()
    s.d_group_map_ptr = t["group_map_ptr"].data_ptr()
    s.d_group_map = t["group_map"].data_ptr()
    s.d_slab_off = t["slab_off"].data_ptr()
    s.d_slab_width = t["slab_width"].data_ptr()
    s.d_slots = t["slots"].data_ptr()
    s.d_values = t["values"].data_ptr()
    s.contract = int(bool(side.contract) and side.precision == "single")
    s.row_group = max(1, int(getattr(info, "row_group", 1) or 1))
    s.chunk_group = max(1, int(side.chunk_group))
    side.staged = s
    plane_slots = -(-int(info.max_group_slots) // 8) * 8
    rec = side.f_dev * element_bytes(side.precision)
    # two stage buffers + two slot->element maps (see spmm.cu)
    side.smem_bytes = int(2 * (plane_slots * rec + 128) + 2 * plane_slots * 4)
    return side


def set_execution(side: DeviceSide, contract: bool, chunk_group: int) -> DeviceSide:
    """Kernel execution knobs of a built side (no rebuild): FFMA
    contraction (single precision, native order only) and the number of
    F-chunks of a tile launched back to back."""
    side.contract = bool(contract) and side.precision == "single"
    side.chunk_group = max(1, int(chunk_group))
    if side.staged is not None:
        side.staged.contract = int(side.contract)
        side.staged.chunk_group = side.chunk_group
    return side


def side_meta(side: DeviceSide) -> dict:
    """Picklable description of a side (everything but the tensor data)."""
    return dict(precision=side.precision, ffactor=side.ffactor, f_dev=side.f_dev,
                n_in=side.n_in, n_out=side.n_out, value_scale_exp=side.value_scale_exp,
                plan_kind=side.plan_kind, contract=side.contract,
                chunk_group=side.chunk_group,
                info={f: getattr(side.info, f) for f in INFO_FIELDS},
                tensors={k: (tuple(v.shape), str(v.dtype).replace("torch.", ""))
                         for k, v in side.tensors.items()})


def side_from_meta(meta: dict, tensors: dict) -> DeviceSide:
    info = _lib.FormatInfo()
    for f, v in meta["info"].items():
        setattr(info, f, v)
    side = DeviceSide(meta["precision"], meta["ffactor"], meta["f_dev"], meta["n_in"],
                      meta["n_out"], meta["value_scale_exp"], info, tensors,
                      plan_kind=meta["plan_kind"], contract=meta.get("contract", False),
                      chunk_group=meta.get("chunk_group", 1))
    return attach(side)
