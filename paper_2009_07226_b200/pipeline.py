"""Operator assembly: the drop-in boundary of the XCT hot path.

Mirrors ``xct.pipeline`` (src/pipeline.py): ``SystemConfig``,
``AssembledSystem`` with ``apply_forward`` / ``apply_adjoint`` /
``num_rows`` / ``num_cols`` / ``kernel_counters`` / ``volume_reports``,
``assemble`` and ``assemble_from_matrix``.  ``cgls_solve`` (solver.py) and
any reference caller use only this surface.

Everything after assembly is device resident: the staged formats of A and
A^T live in HBM and each application runs three of our kernels per call --
chunked max-abs (K7), normalize+cast (K7), staged SpMM with the fused
scale/cast/denormalize epilogue (K6).

P_d > 1 (Hilbert data partitions, src/pipeline.py:104-113) is emulated in
one process here: every rank's partial product runs through K6 and the
partials are reduced in the reference's direct-plan order (owner first,
then senders ascending; src/comm.py:420-472).  The multi-GPU form of the
same decomposition is ``parallel.DomainPartitionedSystem``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from . import _lib, comm, engine, hilbert, matrixstore
from .geometry import ScanGeometry, SystemMatrix, build_system_matrix, device
from .matrixstore import NormalizationState

__all__ = ["SystemConfig", "AssembledSystem", "assemble", "assemble_from_matrix", "ORDERS"]

ORDERS = ("native", "traversal", "reference")


@dataclass(frozen=True)
class SystemConfig:
    """Parallelization and precision knobs (src/pipeline.py:26-47).

    Added for the B200 build (defaults keep the reference's meaning):
      order          "native": image-band / view-range staging with the
                     bank-conflict-free step schedule (sums equal the
                     reference's to rounding); "traversal": the same staging
                     keeping traversal order per ray and ray-id order per
                     voxel (bit-identical to the reference run with
                     stage_capacity_bytes=None, block_partitions=1);
                     "reference": the reference's stage order, bit-identical
                     to the reference's default configuration.
      warps_per_cta  CTA size of the staged SpMM.
      smem_budget    shared-memory bytes per CTA for one load group.
      pieces_per_lane  16-byte pieces of a staged record each lane owns (1, 2
                     or 4; lanes per row = record pieces / this; None = 2,
                     measured fastest with the 64-register K6 at F=16: one
                     lane per row in FP16, two in FP32).
      contract       single precision: one FFMA per entry and slice instead
                     of the reference's multiply-then-add; only with
                     order="native", whose sums already differ from the
                     reference's by rounding (None = on for grouped-row
                     blocks, where it is 20% faster; off for one row per lane
                     set, where it measured 1% slower).
      chunk_group    F-chunks of a CTA tile launched back to back, so their
                     CTAs share the tile's entry stream through L2 (16:
                     measured 1-3% faster than 1 at c2, r01 probe).
      row_group      rows per lane set of K6 (1, 2 or 4; native order,
                     single/mixed): the lanes walk the union of the rows'
                     entries, so each staged record read from shared memory
                     serves row_group rows (2 views x 2 detectors for A,
                     2 x 2 voxels for A^T).
      build          "streamed": never materialize the whole matrix -- the
                     projection format is built per chunk of views, the back
                     projection per band of voxels, from Siddon regenerated
                     on the device ("auto": streamed above STREAM_NNZ).
    ``topology`` and ``comm_strategy`` select the simulated cluster and
    planner of ``volume_reports()`` (byte accounting, `comm.py`); on one
    NVSwitch box the executed exchange has a single level.
    """

    precision: str = "double"
    ffactor: int = 16
    p_b: int = 1
    p_d: int = 1
    tile_size: int = 8
    block_partitions: int = 4
    stage_capacity_bytes: int | None = matrixstore.DEFAULT_STAGE_CAPACITY
    comm_strategy: str = "hierarchical"
    topology: object = None
    workers: int = 1
    order: str = "native"
    warps_per_cta: int = 16
    smem_budget: int = matrixstore.SMEM_BUDGET
    build: str = "auto"
    pieces_per_lane: int | None = None
    contract: bool | None = None
    chunk_group: int = 16
    row_group: int | None = None

    def __post_init__(self):
        if self.precision not in matrixstore.PRECISIONS:
            raise ValueError(f"unknown precision {self.precision!r}")
        if self.comm_strategy not in ("direct", "hierarchical"):
            raise ValueError(f"unknown comm strategy {self.comm_strategy!r}")
        if not 1 <= self.ffactor <= engine.MAX_FFACTOR:
            raise ValueError(f"ffactor must be in [1, {engine.MAX_FFACTOR}]")
        if self.order not in ORDERS:
            raise ValueError(f"unknown order {self.order!r}; expected one of {ORDERS}")
        if self.p_b < 1 or self.p_d < 1:
            raise ValueError("P_b and P_d must be >= 1")
        if self.build not in ("auto", "monolithic", "streamed"):
            raise ValueError(f"unknown build mode {self.build!r}")
        if self.contract and self.order != "native":
            raise ValueError("contract=True changes rounding; it needs order='native'")
        if self.chunk_group < 1:
            raise ValueError("chunk_group must be >= 1")
        if self.row_group not in (None, 1, 2, 4):
            raise ValueError("row_group must be 1, 2 or 4")
        if (self.row_group or 1) > 1 and (self.order != "native" or
                                          self.precision not in ("single", "mixed")):
            raise ValueError("row_group > 1 needs order='native' and single/mixed precision")

    @property
    def smem_budget_effective(self) -> int:
        """Grouped-row blocks run one 512-thread CTA per SM (128 registers a
        thread), so the default budget doubles for them: bigger load groups,
        less padding (measured 5% faster at c2, profiles/r01_probe_c2_smem*)."""
        if self.row_group_effective > 1 and self.smem_budget == matrixstore.SMEM_BUDGET:
            return matrixstore.GROUPED_SMEM_BUDGET
        return self.smem_budget

    @property
    def row_group_effective(self) -> int:
        """None = 4 for native single precision (measured 13-16% faster than
        one row per lane set at c2, profiles/r01_probe_*), 1 otherwise (FP16
        storage: one row per lane is fastest).  The largest of the two
        sides' row groups (side_shape)."""
        if self.row_group is not None:
            return self.row_group
        return 4 if self.order == "native" and self.precision == "single" else 1

    def side_shape(self, kind: str) -> tuple:
        """(row_group, pieces_per_lane) of one operator direction.  Native
        single precision with both unset: A as G=2 units of one lane (each
        lane the whole 64-byte record of 2 rays of adjacent views), A^T as
        G=4 units of two lanes -- measured at c2: A 58.6 -> 52.4 ms, A^T
        46.4 ms vs 50.0 ms with G=2 (profiles/r02_probe_c2_sides.txt).
        Both shapes give 64 rows per warp."""
        if self.row_group is not None:
            return self.row_group, self.pieces_per_lane or 2
        if self.order == "native" and self.precision == "single":
            if self.pieces_per_lane is None and self.ffactor == 16:
                return (2, 4) if kind == "forward" else (4, 2)
            return 4, self.pieces_per_lane or 2
        return 1, self.pieces_per_lane or 2


@dataclass
class _Side:
    """One operator direction: per-rank staged blocks and their maps."""

    blocks: list                 # DeviceSide per rank
    input_elements: list         # global input ids per rank (None = identity)
    footprints: list             # global output ids per rank (None = identity)
    ownership: list              # owned output ids per rank
    num_inputs: int
    num_outputs: int


def configure_execution(sides, config) -> None:
    """Apply the config's kernel execution knobs to every staged block."""
    for side in sides:
        for blk in side.blocks:
            grouped = int(getattr(blk.info, "row_group", 1) or 1) > 1
            c = grouped if config.contract is None else bool(config.contract)
            matrixstore.set_execution(blk, c and config.order == "native", config.chunk_group)


def _rows_per_warp(cfg, row_group: int | None = None, kind: str | None = None) -> int:
    if kind is not None:
        G, ppl = cfg.side_shape(kind)
        return 32 // matrixstore.lanes_for(cfg.ffactor, cfg.precision, ppl) * G
    ppl = cfg.pieces_per_lane or 2
    G = cfg.row_group_effective if row_group is None else row_group
    return 32 // matrixstore.lanes_for(cfg.ffactor, cfg.precision, ppl) * G


def _side_group(cfg, kind: str) -> int:
    return cfg.side_shape(kind)[0]


def _csr_host(matrix):
    if isinstance(matrix, SystemMatrix):
        return matrix.host_csr32()
    return (np.asarray(matrix.indptr, np.int64), np.asarray(matrix.indices, np.int32),
            np.asarray(matrix.values, np.float64))


def _transpose(indptr, indices, values, n_rows, n_cols, alloc=None):
    nnz = len(indices)
    alloc = alloc or (lambda name, n, dt: np.empty(n, dt))
    t_ip = np.empty(n_cols + 1, np.int64)
    t_ix = alloc("t_ix", max(nnz, 1), np.int32)
    t_v = alloc("t_v", max(nnz, 1), np.float64)
    _lib.call("xct_csr_transpose", n_rows, n_cols, indptr.ctypes.data,
              indices.ctypes.data if nnz else None, values.ctypes.data if nnz else None,
              t_ip.ctypes.data, t_ix.ctypes.data, t_v.ctypes.data, _lib.n_threads())
    return t_ip, t_ix[:nnz], t_v[:nnz]


def smem_budget_for(cfg, plan) -> int:
    """Shared memory per CTA: the configured budget, raised for reference
    staging so one whole reference stage fits a (double-buffered) group."""
    if plan.kind != "reference" or cfg.stage_capacity_bytes is None:
        return cfg.smem_budget_effective
    rec = matrixstore.f_dev_for(cfg.ffactor, cfg.precision) * \
        matrixstore.element_bytes(cfg.precision)
    cap = cfg.stage_capacity_bytes // (matrixstore.element_bytes(cfg.precision) * cfg.ffactor)
    return max(cfg.smem_budget, min(2 * cap * rec, matrixstore.SMEM_MAX))


def hilbert_subdomains(geometry, tile_size: int, parts: int):
    """Tomogram and sinogram Hilbert tile segments (src/pipeline.py:104-113)."""
    g = geometry
    tomo = hilbert.decompose(hilbert.TileGrid("tomogram", g.grid_n, g.grid_n, tile_size), parts)
    sino = hilbert.decompose(hilbert.TileGrid("sinogram", g.num_angles, g.num_detector_cols,
                                              tile_size), parts)
    return tomo, sino


def column_block(ip, ix, v, n_rows, n_cols, cols):
    """A[:, cols] over the rows it touches, local ids (src/matrixstore.py:130-148).
    Returns (indptr, local col ids, values, global ids of the footprint rows)."""
    row_of = np.repeat(np.arange(n_rows), np.diff(ip))
    keep = np.zeros(n_cols, bool)
    keep[cols] = True
    sel = keep[ix]
    rows = row_of[sel]
    fp = np.unique(rows)
    lr = np.searchsorted(fp, rows)
    bip = np.concatenate(([0], np.cumsum(np.bincount(lr, minlength=len(fp))))).astype(np.int64)
    bix = np.searchsorted(cols, ix[sel]).astype(np.int32)
    return bip, bix, v[sel], fp


def row_block_transposed(ip, ix, v, rows):
    """transpose(A[rows, :]) over the columns those rows touch
    (src/matrixstore.py:151-165, :189-201).  Returns (indptr, local row
    positions, values, global ids of the footprint columns)."""
    take = (np.concatenate([np.arange(ip[r], ip[r + 1]) for r in rows])
            if len(rows) else np.empty(0, np.int64))
    fp = np.unique(ix[take])
    rip = np.concatenate(([0], np.cumsum(np.diff(ip)[rows]))).astype(np.int64)
    rix = np.searchsorted(fp, ix[take]).astype(np.int32)
    t_ip, t_ix, t_v = _transpose(rip, rix, v[take], len(rows), len(fp))
    return t_ip, t_ix, t_v, fp


def key_shape(geometry, kind):
    """(base B, number of keys) of the device builder's column -> (key,
    coordinate) map: image bands of A (grid_n, grid_n), views of A^T
    (detectors, views)."""
    if kind == "forward":
        return geometry.grid_n, geometry.grid_n
    return geometry.num_detector_cols, geometry.num_angles


def device_side_from_csr(geometry, cfg, plan, ip, ix, v, n_rows, n_cols, exp, budget, dev):
    """K5 on the device from a host CSR (uploaded); None if the device
    builder declines (the caller falls back to the host builder)."""
    import torch
    b, nk = key_shape(geometry, plan.kind)
    d_ip = torch.from_numpy(np.ascontiguousarray(ip, np.int64)).to(dev)
    d_ix = torch.from_numpy(np.ascontiguousarray(ix, np.int32)).to(dev)
    d_v = torch.from_numpy(np.ascontiguousarray(v, np.float64)).to(dev)
    try:
        part = matrixstore.build_format_device(d_ip, d_ix, d_v, n_rows, n_cols, plan,
                                               cfg.precision, cfg.ffactor, exp, budget,
                                               cfg.order == "native", b, nk, dev)
    except matrixstore.DeviceBuildUnsupported as e:
        _log(f"device format build declined ({e}); host builder")
        return None
    return matrixstore.combine_device_parts([part], cfg.precision, cfg.ffactor, n_cols, n_rows,
                                            exp, dev)


class AssembledSystem:
    """Distributed forward/adjoint operator over one batch group's slices
    (src/pipeline.py:64-210), device resident."""

    def __init__(self, matrix, config: SystemConfig, geometry: ScanGeometry | None = None):
        self.matrix = matrix
        self.config = config
        self.geometry = geometry
        self.device = device()
        cfg = config
        if cfg.precision in ("half", "mixed"):
            vals = getattr(matrix, "d_values", None)
            self.value_scale_exp = matrixstore.half_rescale_exponent(
                vals if vals is not None else np.asarray(matrix.values, np.float64))
        else:
            self.value_scale_exp = 0
        ip, ix, v = _csr_host(matrix)
        n_rows, n_cols = int(matrix.num_rows), int(matrix.num_cols)
        if cfg.p_d == 1:
            self.forward = self._single_side(ip, ix, v, n_rows, n_cols, "forward")
            t_ip, t_ix, t_v = _transpose(ip, ix, v, n_rows, n_cols)
            self.adjoint = self._single_side(t_ip, t_ix, t_v, n_cols, n_rows, "adjoint")
        else:
            if geometry is None:
                raise ValueError("data parallelism beyond P_d=1 needs a scan geometry")
            self._build_partitioned(ip, ix, v, n_rows, n_cols)
        configure_execution((self.forward, self.adjoint), cfg)

    @classmethod
    def from_sides(cls, matrix, config: SystemConfig, geometry, forward_block, adjoint_block,
                   value_scale_exp: int) -> "AssembledSystem":
        """Wrap already-built device sides (e.g. received by broadcast)."""
        self = cls.__new__(cls)
        self.matrix, self.config, self.geometry = matrix, config, geometry
        self.device = device()
        self.value_scale_exp = value_scale_exp
        n_rows, n_cols = int(matrix.num_rows), int(matrix.num_cols)
        self.forward = _Side([forward_block], [None], [None], [np.arange(n_rows)], n_cols, n_rows)
        self.adjoint = _Side([adjoint_block], [None], [None], [np.arange(n_cols)], n_rows, n_cols)
        configure_execution((self.forward, self.adjoint), config)
        return self

    # -- construction ---------------------------------------------------------

    def _plan(self, ip, ix, n_rows, n_cols, kind):
        cfg, g = self.config, self.geometry
        rw = _rows_per_warp(cfg, kind=kind)
        if kind == "forward":
            if cfg.order == "reference" or g is None:
                return matrixstore.reference_plan(ip, ix, n_rows, n_cols, cfg.block_partitions,
                                                  cfg.stage_capacity_bytes, cfg.ffactor,
                                                  cfg.precision, _rows_per_warp(cfg, 1),
                                                  cfg.warps_per_cta)
            plan = matrixstore.forward_plan(g.num_angles, g.grid_n, rw, cfg.warps_per_cta,
                                            row_group=_side_group(cfg, "forward"))
            return matrixstore.assign_forward_regimes(plan, g.angles, g.grid_n)
        # adjoint: every per-voxel order keyed by ascending ray id is the
        # reference order (src/matrixstore.py:189-201 sorts entries by ray)
        if g is not None and n_rows == g.num_voxels and n_cols == g.num_rays:
            return matrixstore.adjoint_plan(g.num_angles, g.grid_n, rw, cfg.warps_per_cta,
                                            row_group=_side_group(cfg, "adjoint"))
        return matrixstore.row_block_plan(n_rows, n_cols, rw, cfg.warps_per_cta,
                                          row_group=_side_group(cfg, "adjoint"))

    def _budget(self, plan) -> int:
        return smem_budget_for(self.config, plan)

    def _single_side(self, ip, ix, v, n_rows, n_cols, kind) -> _Side:
        cfg = self.config
        plan = self._plan(ip, ix, n_rows, n_cols, kind)
        blk = None
        if matrixstore.device_build_supported(plan, cfg.precision):
            blk = device_side_from_csr(self.geometry, cfg, plan, ip, ix, v, n_rows, n_cols,
                                       self.value_scale_exp, self._budget(plan), self.device)
        if blk is None:
            blk = matrixstore.build_device_side(ip, ix, v, n_rows, n_cols, plan, cfg.precision,
                                                cfg.ffactor, self.value_scale_exp,
                                                self._budget(plan), self.device,
                                                schedule=cfg.order == "native")
        ident = np.arange(n_rows)
        return _Side([blk], [None], [None], [ident], n_cols, n_rows)

    def _build_partitioned(self, ip, ix, v, n_rows, n_cols):
        cfg, g = self.config, self.geometry
        tomo, sino = hilbert_subdomains(g, cfg.tile_size, cfg.p_d)
        self.tomogram_subdomains, self.sinogram_subdomains = tomo, sino
        rw = _rows_per_warp(cfg, 1)

        def build(bip, bix, bv, nr, nc):
            plan = matrixstore.reference_plan(bip, bix, nr, nc, cfg.block_partitions,
                                              cfg.stage_capacity_bytes, cfg.ffactor,
                                              cfg.precision, rw, cfg.warps_per_cta)
            return matrixstore.build_device_side(bip, bix, bv, nr, nc, plan, cfg.precision,
                                                 cfg.ffactor, self.value_scale_exp,
                                                 self._budget(plan), self.device)

        f_blocks, f_fp, a_blocks, a_fp = [], [], [], []
        for sub in tomo:
            bip, bix, bv, fp = column_block(ip, ix, v, n_rows, n_cols, sub.elements)
            f_blocks.append(build(bip, bix, bv, len(fp), len(sub.elements)))
            f_fp.append(fp)
        for sub in sino:
            t_ip, t_ix, t_v, fp = row_block_transposed(ip, ix, v, sub.elements)
            a_blocks.append(build(t_ip, t_ix, t_v, len(fp), len(sub.elements)))
            a_fp.append(fp)
        self.forward = _Side(f_blocks, [s.elements for s in tomo], f_fp,
                             [s.elements for s in sino], n_cols, n_rows)
        self.adjoint = _Side(a_blocks, [s.elements for s in sino], a_fp,
                             [s.elements for s in tomo], n_rows, n_cols)

    # -- application ------------------------------------------------------------

    @property
    def num_cols(self) -> int:
        return int(self.matrix.num_cols)

    @property
    def num_rows(self) -> int:
        return int(self.matrix.num_rows)

    def apply_forward(self, x):
        """Projection of (num_cols,) or (num_cols, slices) data; returns
        (values, [NormalizationState per F-chunk]) (src/pipeline.py:141-174)."""
        return self._apply(self.forward, x)

    def apply_adjoint(self, y):
        return self._apply(self.adjoint, y)

    def _apply(self, side: _Side, data):
        import torch
        is_np = not isinstance(data, torch.Tensor)
        arr = np.asarray(data) if is_np else data
        squeeze = arr.ndim == 1
        if arr.shape[0] != side.num_inputs:
            raise ValueError(f"operator expects {side.num_inputs} input elements, "
                             f"got {arr.shape[0]}")
        dev = self.device
        X = torch.as_tensor(arr, device=dev)
        if X.dtype not in (torch.float32, torch.float64):
            X = X.to(torch.float64)
        X = X.reshape(X.shape[0], -1).contiguous()
        S = int(X.shape[1])
        cfg = self.config
        F = cfg.ffactor
        out_dtype = torch.float64 if cfg.precision == "double" else torch.float32
        out = torch.empty((side.num_outputs, S), dtype=out_dtype, device=dev)
        states = []
        if S == 0:
            res = out.cpu().numpy() if is_np else out
            return (res[:, 0] if squeeze else res), states
        n_chunks = -(-S // F)
        st = _lib.stream_handle(dev)
        in64 = int(X.dtype == torch.float64)
        maxbits = torch.zeros(n_chunks, dtype=torch.int64, device=dev)
        _lib.call("xct_chunk_maxabs", X.data_ptr(), in64, X.shape[0], S, S, F, n_chunks,
                  maxbits.data_ptr(), st)
        factors = matrixstore._peaks_to_factors(maxbits)
        states = [NormalizationState(factor=f, mode=cfg.precision) for f in factors]
        fac = torch.tensor(factors, dtype=torch.float64, device=dev)
        blk0 = side.blocks[0]
        sd = {"double": torch.float64, "single": torch.float32}.get(cfg.precision, torch.float16)
        if len(side.blocks) == 1 and side.input_elements[0] is None:
            xin = torch.empty((n_chunks, side.num_inputs, blk0.f_dev), dtype=sd, device=dev)
            _lib.call("xct_normalize", X.data_ptr(), in64, X.shape[0], S, S, F, n_chunks,
                      blk0.f_dev, fac.data_ptr(), _lib.PREC_CODE[cfg.precision],
                      xin.data_ptr(), st)
            engine.apply_side(blk0, xin, out, row_stride=S, chunk_stride=F, valid_cols=S,
                              ffactor_out=F, factors=fac, stream=st)
        else:
            self._apply_partitioned(side, X, S, F, n_chunks, fac, sd, out, st)
        res = out.cpu().numpy() if is_np else out
        return (res[:, 0] if squeeze else res), states

    def _apply_partitioned(self, side, X, S, F, n_chunks, fac, sd, out, st):
        """Per-rank partials, then the direct-plan reduction order."""
        import torch
        cfg, dev = self.config, self.device
        in64 = int(X.dtype == torch.float64)
        cd = {"double": torch.float64, "half": torch.float16}.get(cfg.precision, torch.float32)
        f_dev = side.blocks[0].f_dev
        xin = torch.empty((n_chunks, side.num_inputs, f_dev), dtype=sd, device=dev)
        _lib.call("xct_normalize", X.data_ptr(), in64, X.shape[0], S, S, F, n_chunks, f_dev,
                  fac.data_ptr(), _lib.PREC_CODE[cfg.precision], xin.data_ptr(), st)
        pdt = torch.float64 if cfg.precision == "double" else torch.float32
        parts = []
        for blk, inp in zip(side.blocks, side.input_elements):
            xp = xin[:, torch.as_tensor(inp, device=dev)].contiguous()
            pr = torch.empty((blk.n_out, n_chunks * F), dtype=pdt, device=dev)
            engine.apply_side(blk, xp, pr, row_stride=n_chunks * F, chunk_stride=F,
                              valid_cols=n_chunks * F, ffactor_out=F, factors=None, stream=st)
            parts.append(pr.to(cd))
        if cfg.comm_strategy == "hierarchical":
            total = self._replay_hierarchical(side, parts, cd, n_chunks * F)
        else:
            total = torch.zeros((side.num_outputs, n_chunks * F), dtype=cd, device=dev)
            cols = n_chunks * F
            for q, own in enumerate(side.ownership):
                keep = np.zeros(side.num_outputs, dtype=bool)
                keep[np.asarray(own)] = True
                for s in [q] + [s for s in range(len(parts)) if s != q]:
                    fp = np.asarray(side.footprints[s])
                    sel = np.nonzero(keep[fp])[0]
                    if len(sel) == 0:
                        continue
                    if cd == torch.float16:          # K10 moves f32/f64 rows only
                        idx = torch.as_tensor(sel, device=dev)
                        total[torch.as_tensor(fp[sel], device=dev)] += parts[s][idx]
                        continue
                    # K10: gather the rows this owner takes from rank s, add
                    # them at their output positions (owner first, then the
                    # senders ascending: the direct plan's order)
                    f64 = int(cd == torch.float64)
                    d_sel = torch.as_tensor(sel.astype(np.int32), device=dev)
                    d_pos = torch.as_tensor(fp[sel].astype(np.int32), device=dev)
                    buf = torch.empty((len(sel), cols), dtype=cd, device=dev)
                    _lib.call("xct_gather_rows", parts[s].data_ptr(), parts[s].shape[0],
                              d_sel.data_ptr(), len(sel), 1, cols, f64, buf.data_ptr(), st)
                    _lib.call("xct_accumulate_rows", total.data_ptr(), side.num_outputs,
                              buf.data_ptr(), d_pos.data_ptr(), len(sel), 1, cols, f64, st)
        odt = torch.float64 if cfg.precision == "double" else torch.float32
        f_cols = fac.to(odt).repeat_interleave(F)[None, :]
        res = total.to(odt) * f_cols
        out.copy_(res[:, :S])

    def _replay_hierarchical(self, side, parts, cd, cols):
        """The reference's execute_plan (src/comm.py:420-472) for the
        hierarchical plan of this side (socket, node, then global level over
        the configured topology): every level's transfers in sorted (sender,
        receiver) order, the receiver adding each arriving contribution to
        what it holds -- the same summation order as the reference, so
        order="reference" results stay bit-identical with its default
        comm_strategy.  (One process; dense per-process buffers, a
        small-problem emulation path.)"""
        import torch
        dev, cfg = self.device, self.config
        key = "projection" if side is self.forward else "backprojection"
        plans = getattr(self, "_hier_plans", None)
        if plans is None:
            plans = self._hier_plans = {}
        if key not in plans:
            topo = cfg.topology if cfg.topology is not None else comm.default_topology()
            placement = comm.map_partitions(cfg.p_b, cfg.p_d, topo)
            eb = matrixstore.element_bytes(cfg.precision)
            fps = {p: np.asarray(fp) for p, fp in enumerate(side.footprints)}
            own = {q: np.asarray(o) for q, o in enumerate(side.ownership)}
            plans[key] = comm.plan_hierarchical(fps, own, placement, ffactor=cfg.ffactor,
                                                elem_bytes=eb)[0]
        plan = plans[key]
        n = side.num_outputs
        P = max(len(parts), len(side.ownership))
        vals = torch.zeros((P, n, cols), dtype=cd, device=dev)
        has = torch.zeros((P, n), dtype=torch.bool, device=dev)
        for p, part in enumerate(parts):
            rows = torch.as_tensor(np.asarray(side.footprints[p]), device=dev)
            vals[p, rows] = part
            has[p, rows] = True
        for level in plan.levels:
            for (s_, r_) in sorted(level.transfers):
                e = torch.as_tensor(np.asarray(level.transfers[(s_, r_)], np.int64), device=dev)
                contrib = vals[s_, e]
                has[s_, e] = False
                prior = has[r_, e]
                vals[r_, e] = torch.where(prior[:, None], vals[r_, e] + contrib, contrib)
                has[r_, e] = True
        total = torch.zeros((n, cols), dtype=cd, device=dev)
        for q, own in enumerate(side.ownership):
            o = torch.as_tensor(np.asarray(own, np.int64), device=dev)
            total[o] = torch.where(has[q, o][:, None], vals[q, o], total[o])
        return total

    # -- reporting ----------------------------------------------------------------

    def kernel_counters(self) -> engine.KernelCounters:
        """Aggregate work counters for one forward application."""
        return engine.kernel_counters(self.forward.blocks)

    def volume_reports(self) -> dict:
        """Per-level exchange byte accounting, `comm.VolumeReport` per side,
        equal to the reference's (src/pipeline.py:115-124, :192-194): the
        planner named by ``comm_strategy`` over ``topology`` (default: the
        reference's 4 x 2 x 3 cluster).  Computed on first call, not at
        assembly, because the simulated placement may not fit a P_b that the
        B200 slice batch runs (the reference raises then, here this call does)."""
        if getattr(self, "_volume_reports", None) is None:
            cfg = self.config
            topo = cfg.topology if cfg.topology is not None else comm.default_topology()
            placement = comm.map_partitions(cfg.p_b, cfg.p_d, topo)
            planner = (comm.plan_hierarchical if cfg.comm_strategy == "hierarchical"
                       else comm.plan_direct)
            eb = matrixstore.element_bytes(cfg.precision)
            out = {}
            for name, side in (("projection", self.forward), ("backprojection", self.adjoint)):
                fps = {p: (fp if fp is not None else self._nonempty_outputs(name))
                       for p, fp in enumerate(side.footprints)}
                own = {q: np.asarray(o) for q, o in enumerate(side.ownership)}
                out[name] = planner(fps, own, placement, ffactor=cfg.ffactor,
                                    elem_bytes=eb)[1]
            self._volume_reports = out
        return self._volume_reports

    def _nonempty_outputs(self, name) -> np.ndarray:
        """P_d = 1 footprint: output elements with at least one entry
        (src/matrixstore.py:130-148 drops empty rows / untouched columns)."""
        m = self.matrix
        n_rows, n_cols = int(m.num_rows), int(m.num_cols)
        rec = getattr(self, "_nonempty", None)
        if rec is not None:                 # streamed build: recorded while building
            return rec[name]
        ip, ix = getattr(m, "indptr", None), getattr(m, "indices", None)
        if ip is None or ix is None:
            raise ValueError("volume_reports needs the operator's non-empty rows/columns")
        if name == "projection":
            return np.flatnonzero(np.diff(np.asarray(ip)) > 0)
        return np.unique(np.asarray(ix))

    def hbm_bytes(self) -> int:
        return sum(b.hbm_bytes() for s in (self.forward, self.adjoint) for b in s.blocks)


STREAM_NNZ = 6e8        # auto mode streams operators larger than this


def _streamable(geometry, config) -> bool:
    if config.p_d != 1 or config.order == "reference" or config.build == "monolithic":
        return False
    if config.build == "streamed":
        return True
    return 1.2 * geometry.num_angles * geometry.grid_n ** 2 > STREAM_NNZ


def assemble(geometry: ScanGeometry, config: SystemConfig) -> AssembledSystem:
    """Build the device operator for a scan geometry (matrix memoized)."""
    if _streamable(geometry, config):
        return StreamedAssembly(geometry, config).run()
    return AssembledSystem(build_system_matrix(geometry), config, geometry=geometry)


def assemble_from_matrix(matrix, config: SystemConfig | None = None) -> AssembledSystem:
    """Wrap an arbitrary compressed-row operator (single data process)."""
    config = config or SystemConfig(p_d=1)
    if config.p_d != 1:
        config = replace(config, p_d=1)
    return AssembledSystem(matrix, config, geometry=None)


def _log(msg):
    import os
    import sys
    if os.environ.get("XCT_VERBOSE"):
        print(f"[xct] {msg}", file=sys.stderr, flush=True)


class _Timer:
    def __init__(self):
        import time
        self.t, self.acc = time.perf_counter(), {}

    def lap(self, key):
        import time
        now = time.perf_counter()
        self.acc[key] = self.acc.get(key, 0.0) + now - self.t
        self.t = now


def Plan_probe(cfg):
    """A plan-shaped probe of what the streamed build would run (plan kind
    and row group) for device_build_supported."""
    return matrixstore.Plan(np.zeros((0, 1), np.int32), np.zeros((1, 1), np.int32),
                            np.zeros(0, np.int32), 1, "forward", cfg.row_group_effective)


class StreamedAssembly:
    """Operator build that never holds the whole matrix (needed at 2048^2 x
    2048 views, 1.03e10 entries): Siddon is regenerated on the device per
    chunk of views; the projection format is built chunk by chunk, the back
    projection format band of voxel rows by band (each band's entries are
    the column-restricted chunks, transposed on the host).  Per-row orders
    and load groups are exactly those of the monolithic build."""

    CHUNK_NNZ = 4e8          # entries per Siddon chunk on the device / host
    BAND_NNZ = 1.2e9         # entries per back-projection band on the host

    def __init__(self, geometry: ScanGeometry, config: SystemConfig):
        self.g, self.cfg = geometry, config
        self.dev = device()
        self.rw = _rows_per_warp(config, kind="forward")
        self.rw_a = _rows_per_warp(config, kind="adjoint")
        self._pool = {}

    def _buf(self, name, n, dtype, pinned=False):
        """Reusable host buffer (page-locked for the D2H targets): fresh
        allocations per chunk would pay the page faults again every time."""
        import torch
        dt = np.dtype(dtype)
        need = int(n) * dt.itemsize
        t = self._pool.get(name)
        if t is None or t.numel() < need:
            self._pool.pop(name, None)
            t = torch.empty(int(need * 1.05) + 64, dtype=torch.uint8, pin_memory=pinned)
            self._pool[name] = t
        return t[:need].numpy().view(dt)

    def _d2h(self, name, t):
        """Device tensor -> pooled host array (through the pinned staging;
        page-locking GBs up front costs more than it saves)."""
        import torch
        out = self._buf(name, t.numel(), torch.empty((), dtype=t.dtype).numpy().dtype)
        return _lib.to_host(t, out=out)

    def _chunks(self, align: int):
        g = self.g
        per = max(1, int(self.CHUNK_NNZ // (1.2 * g.grid_n ** 2)))
        per = max(align, per // align * align)
        return [(k, min(k + per, g.num_angles)) for k in range(0, g.num_angles, per)]

    def _siddon(self, k0, k1):
        from .geometry import siddon_csr
        return siddon_csr(self.g, k0, k1, self.dev)

    def _exponent(self, chunks) -> int:
        """half_rescale_exponent over the whole matrix without holding it:
        exact binade histogram of the positive lengths, then the two middle
        values when they straddle a binade (numpy median: their mean)."""
        import torch
        hist = torch.zeros(2048, dtype=torch.int64, device=self.dev)
        st = _lib.stream_handle(self.dev)
        for k0, k1 in chunks:
            _, _, v = self._siddon(k0, k1)
            _lib.call("xct_binade_hist", v.data_ptr(), v.numel(), hist.data_ptr(), st)
        n = int(hist.sum())
        if n == 0:
            return 0
        cum = torch.cumsum(hist, 0).cpu().numpy()
        lo_rank, hi_rank = (n - 1) // 2, n // 2                 # 0-based middle ranks
        b_lo = int(np.searchsorted(cum, lo_rank, side="right"))
        b_hi = int(np.searchsorted(cum, hi_rank, side="right"))
        if b_lo == b_hi:
            return -(b_lo - 1023)
        # two middle values in adjacent binades: largest of b_lo, smallest of b_hi
        big, small = -math.inf, math.inf
        for k0, k1 in chunks:
            _, _, v = self._siddon(k0, k1)
            e = (v.view(torch.int64) >> 52)
            a = v[(v > 0) & (e == b_lo)]
            b = v[(v > 0) & (e == b_hi)]
            if a.numel():
                big = max(big, float(a.max()))
            if b.numel():
                small = min(small, float(b.min()))
        return -int(math.floor(math.log2((big + small) / 2.0)))

    def _forward(self, exp):
        import torch
        cfg, g = self.cfg, self.g
        n = g.grid_n
        Gf = _side_group(cfg, "forward")
        ta = matrixstore.forward_tile_height(n, self.rw, cfg.warps_per_cta, Gf, g.num_angles)
        parts = []
        tm = _Timer()
        for k0, k1 in self._chunks(ta):
            plan = matrixstore.forward_plan(g.num_angles, n, self.rw, cfg.warps_per_cta, k0, k1,
                                            row_group=Gf)
            plan = matrixstore.assign_forward_regimes(plan, g.angles, n)
            base = k0 * n
            plan.cta_rows = np.where(plan.cta_rows >= 0, plan.cta_rows - base, -1).astype(np.int32)
            tm.lap("plan")
            ip, ix, v = self._siddon(k0, k1)
            self.ray_hit[k0 * n:k1 * n] = torch.diff(ip) > 0
            _lib.call("xct_csr_col_counts", ip.data_ptr(), ix.data_ptr(), (k1 - k0) * n, 0,
                      g.num_voxels, self.col_counts.data_ptr(), _lib.stream_handle(self.dev))
            ip, ix, v = self._d2h("f_ip", ip), self._d2h("f_ix", ix), self._d2h("f_v", v)
            tm.lap("siddon+d2h")
            hf = matrixstore.build_format(ip, ix, v, (k1 - k0) * n, g.num_voxels, plan,
                                          cfg.precision, cfg.ffactor, exp, cfg.smem_budget_effective,
                                          schedule=cfg.order == "native")
            tm.lap("format")
            hf.cta_rows = np.where(hf.cta_rows >= 0, hf.cta_rows + base, -1).astype(np.int32)
            parts.append(hf)
            self.nnz += int(hf.info["nnz"])
        side = matrixstore.upload_format(parts, cfg.precision, cfg.ffactor, g.num_voxels,
                                         g.num_rays, exp, self.dev)
        tm.lap("upload")
        _log(f"forward build {tm.acc}")
        return side

    def _adjoint(self, exp, chunks):
        import torch
        cfg, g = self.cfg, self.g
        n, R = g.grid_n, g.num_rays
        Ga = _side_group(cfg, "adjoint")
        tz = matrixstore.adjoint_tile_height(n, self.rw_a, cfg.warps_per_cta, Ga)
        per = max(1, int(self.BAND_NNZ // (1.2 * g.num_angles * n)))
        per = max(tz, per // tz * tz)
        st = _lib.stream_handle(self.dev)
        parts = []
        tm = _Timer()
        for z0 in range(0, n, per):
            z1 = min(n, z0 + per)
            lo, hi = z0 * n, z1 * n
            # the band's entries go straight from the pinned staging into
            # one host CSR (capacity from the ~1.27 rays/view/voxel of a
            # parallel beam; grown if ever short)
            counts = []
            cap = int((hi - lo) * g.num_angles * 1.45) + 1024
            bix, bv, at = self._buf("a_ix", cap, np.int32), self._buf("a_v", cap, np.float64), 0
            for k0, k1 in chunks:
                ip, ix, v = self._siddon(k0, k1)
                rows = (k1 - k0) * n
                cnt = torch.empty(rows, dtype=torch.int64, device=self.dev)
                _lib.call("xct_csr_filter_cols", ip.data_ptr(), ix.data_ptr(), v.data_ptr(),
                          rows, lo, hi, cnt.data_ptr(), None, None, None, st)
                optr = torch.zeros(rows + 1, dtype=torch.int64, device=self.dev)
                torch.cumsum(cnt, 0, out=optr[1:])
                m = int(optr[-1])
                oi = torch.empty(max(m, 1), dtype=torch.int32, device=self.dev)
                ov = torch.empty(max(m, 1), dtype=torch.float64, device=self.dev)
                _lib.call("xct_csr_filter_cols", ip.data_ptr(), ix.data_ptr(), v.data_ptr(),
                          rows, lo, hi, None, optr.data_ptr(), oi.data_ptr(), ov.data_ptr(), st)
                if at + m > cap:
                    cap = max(at + m, int(cap * 1.5))
                    bix, bv = bix[:at].copy(), bv[:at].copy()
                    bix2, bv2 = self._buf("a_ix", cap, np.int32), self._buf("a_v", cap, np.float64)
                    bix2[:at], bv2[:at] = bix, bv
                    bix, bv = bix2, bv2
                counts.append(_lib.to_host(cnt))
                _lib.to_host(oi[:m], out=bix[at:at + m])
                _lib.to_host(ov[:m], out=bv[at:at + m])
                at += m
            tm.lap("siddon+filter+d2h")
            bip = np.zeros(R + 1, np.int64)
            np.cumsum(np.concatenate(counts), out=bip[1:])
            bix, bv = bix[:at], bv[:at]
            del counts
            tm.lap("concat")
            t_ip, t_ix, t_v = _transpose(bip, bix, bv, R, hi - lo, alloc=self._buf)
            del bip, bix, bv
            tm.lap("transpose")
            plan = matrixstore.adjoint_plan(g.num_angles, n, self.rw_a, cfg.warps_per_cta, z0, z1,
                                            row_group=Ga)
            plan.cta_rows = np.where(plan.cta_rows >= 0, plan.cta_rows - lo, -1).astype(np.int32)
            tm.lap("plan")
            hf = matrixstore.build_format(t_ip, t_ix, t_v, hi - lo, R, plan, cfg.precision,
                                          cfg.ffactor, exp, cfg.smem_budget_effective,
                                          schedule=cfg.order == "native")
            tm.lap("format")
            hf.cta_rows = np.where(hf.cta_rows >= 0, hf.cta_rows + lo, -1).astype(np.int32)
            parts.append(hf)
        side = matrixstore.upload_format(parts, cfg.precision, cfg.ffactor, R, g.num_voxels,
                                         exp, self.dev)
        tm.lap("upload")
        _log(f"adjoint build {tm.acc}")
        return side

    # --- K4/K5 on the device ------------------------------------------------
    BAND_NNZ_DEV = 2.5e9     # entries of one device A^T band (12 B each)

    def _device_ok(self) -> bool:
        cfg = self.cfg
        probe = Plan_probe(cfg)
        return matrixstore.device_build_supported(probe, cfg.precision)

    def _forward_device(self, exp, col_counts):
        """Projection format on the device, chunk of views by chunk; also
        counts each voxel's entries (the back projection's row lengths)."""
        import torch
        cfg, g = self.cfg, self.g
        n = g.grid_n
        ta = matrixstore.forward_tile_height(n, self.rw, cfg.warps_per_cta, 1, g.num_angles)
        st = _lib.stream_handle(self.dev)
        parts = []
        tm = _Timer()
        for k0, k1 in self._chunks(ta):
            plan = matrixstore.forward_plan(g.num_angles, n, self.rw, cfg.warps_per_cta, k0, k1,
                                            row_group=1)
            plan = matrixstore.assign_forward_regimes(plan, g.angles, n)
            base = k0 * n
            plan.cta_rows = np.where(plan.cta_rows >= 0, plan.cta_rows - base, -1).astype(np.int32)
            tm.lap("plan")
            ip, ix, v = self._siddon(k0, k1)
            rows = (k1 - k0) * n
            _lib.call("xct_csr_col_counts", ip.data_ptr(), ix.data_ptr(), rows, 0, g.num_voxels,
                      col_counts.data_ptr(), st)
            self.ray_hit[k0 * n:k1 * n] = torch.diff(ip) > 0
            tm.lap("siddon")
            part = matrixstore.build_format_device(ip, ix, v, rows, g.num_voxels, plan,
                                                   cfg.precision, cfg.ffactor, exp,
                                                   cfg.smem_budget_effective,
                                                   cfg.order == "native", n, n, self.dev)
            cr = part.tensors["cta_rows"]
            part.tensors["cta_rows"] = torch.where(cr >= 0, cr + base, cr)
            parts.append(part)
            self.nnz += int(part.info["nnz"])
            del ip, ix, v
            tm.lap("format")
        side = matrixstore.combine_device_parts(parts, cfg.precision, cfg.ffactor, g.num_voxels,
                                                g.num_rays, exp, self.dev)
        torch.cuda.synchronize(self.dev)
        tm.lap("combine")
        _log(f"forward build (device) {tm.acc}")
        return side

    def _adjoint_device(self, exp, chunks, col_counts):
        """Back projection format on the device, band of voxel rows by band:
        the band's A^T rows (ascending ray id) by the device transpose, then
        device K5."""
        import torch
        cfg, g = self.cfg, self.g
        n, R = g.grid_n, g.num_rays
        tz = matrixstore.adjoint_tile_height(n, self.rw, cfg.warps_per_cta, 1)
        st = _lib.stream_handle(self.dev)
        per_row = col_counts.view(n, n).sum(1).cpu().numpy()      # entries per image row
        bands, z0 = [], 0
        while z0 < n:
            z1, acc = z0, 0
            while z1 < n and (z1 == z0 or acc + per_row[z1:z1 + tz].sum() <= self.BAND_NNZ_DEV):
                acc += per_row[z1:z1 + tz].sum()
                z1 = min(n, z1 + tz)
            bands.append((z0, z1))
            z0 = z1
        parts = []
        tm = _Timer()
        for z0, z1 in bands:
            lo, hi = z0 * n, z1 * n
            nb = hi - lo
            t_ip = torch.zeros(nb + 1, dtype=torch.int64, device=self.dev)
            torch.cumsum(col_counts[lo:hi], 0, out=t_ip[1:])
            m = int(t_ip[-1].item())
            t_rows = torch.empty(max(m, 1), dtype=torch.int32, device=self.dev)
            t_vals = torch.empty(max(m, 1), dtype=torch.float64, device=self.dev)
            cursor = torch.zeros(nb, dtype=torch.int32, device=self.dev)
            prev = torch.zeros(nb, dtype=torch.int32, device=self.dev)
            for k0, k1 in chunks:
                ip, ix, v = self._siddon(k0, k1)
                _lib.call("xct_csr_transpose_band", ip.data_ptr(), ix.data_ptr(), v.data_ptr(),
                          (k1 - k0) * n, k0 * n, 32 * n, lo, hi, t_ip.data_ptr(),
                          cursor.data_ptr(), prev.data_ptr(), t_rows.data_ptr(),
                          t_vals.data_ptr(), st)
                del ip, ix, v
            tm.lap("siddon+transpose")
            plan = matrixstore.adjoint_plan(g.num_angles, n, self.rw, cfg.warps_per_cta, z0, z1,
                                            row_group=1)
            plan.cta_rows = np.where(plan.cta_rows >= 0, plan.cta_rows - lo, -1).astype(np.int32)
            part = matrixstore.build_format_device(t_ip, t_rows, t_vals, nb, R, plan,
                                                   cfg.precision, cfg.ffactor, exp,
                                                   cfg.smem_budget_effective,
                                                   cfg.order == "native",
                                                   g.num_detector_cols, g.num_angles, self.dev)
            cr = part.tensors["cta_rows"]
            part.tensors["cta_rows"] = torch.where(cr >= 0, cr + lo, cr)
            parts.append(part)
            del t_ip, t_rows, t_vals, cursor, prev
            tm.lap("format")
        side = matrixstore.combine_device_parts(parts, cfg.precision, cfg.ffactor, R,
                                                g.num_voxels, exp, self.dev)
        torch.cuda.synchronize(self.dev)
        tm.lap("combine")
        _log(f"adjoint build (device) {tm.acc}")
        return side

    def run(self) -> AssembledSystem:
        import torch
        from .parallel import MatrixInfo
        cfg, g = self.cfg, self.g
        ta = matrixstore.forward_tile_height(g.grid_n, self.rw, cfg.warps_per_cta,
                                             _side_group(cfg, "forward"), g.num_angles)
        chunks = self._chunks(ta)
        exp = self._exponent(chunks) if cfg.precision in ("half", "mixed") else 0
        self.nnz = 0
        # outputs with at least one entry (the reference's footprints drop
        # empty rays and untouched voxels, src/matrixstore.py:130-148)
        self.ray_hit = torch.zeros(g.num_rays, dtype=torch.bool, device=self.dev)
        self.col_counts = torch.zeros(g.num_voxels, dtype=torch.int64, device=self.dev)
        if self._device_ok():
            try:
                fwd = self._forward_device(exp, self.col_counts)
                adj = self._adjoint_device(exp, chunks, self.col_counts)
                # hand the build's cached blocks (fill scratch, band buffers)
                # back, so the solver's large vectors do not meet a
                # fragmented cache next to a 93 GB operator
                torch.cuda.empty_cache()
                info = MatrixInfo(g.num_rays, g.num_voxels, self.nnz, g.num_angles,
                                  g.num_detector_cols)
                return self._attach(AssembledSystem.from_sides(info, cfg, g, fwd, adj, exp))
            except matrixstore.DeviceBuildUnsupported as e:
                _log(f"device format build declined ({e}); host builder")
                self.nnz = 0
                torch.cuda.empty_cache()
        fwd = self._forward(exp)
        self._pool.clear()
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        adj = self._adjoint(exp, chunks)
        self._pool.clear()
        torch.cuda.empty_cache()
        info = MatrixInfo(g.num_rays, g.num_voxels, self.nnz, g.num_angles, g.num_detector_cols)
        return self._attach(AssembledSystem.from_sides(info, cfg, g, fwd, adj, exp))

    def _attach(self, system):
        system._nonempty = {
            "projection": self.ray_hit.nonzero().reshape(-1).cpu().numpy(),
            "backprojection": (self.col_counts > 0).nonzero().reshape(-1).cpu().numpy()}
        return system
