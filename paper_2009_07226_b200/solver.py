"""CGLS reconstruction on the device.

Mirrors ``xct.solver`` (src/solver.py): SolveConfig, SolveResult,
SolverDivergence, early_stop, residual_curve_report and cgls_solve, with
the reference's exact scalar and cast sequence:

  * scalars (alpha, beta, norms) are float64 host floats, cast to the work
    dtype before use (src/solver.py:172-185);
  * vector updates are one multiply then one add (two roundings) in the
    work dtype -- K8 ``xct_axpy``;
  * half/mixed keep x, r, p as fp16 payload + max-abs factor
    (_VectorStore, src/solver.py:84-108): a max pass, then a store pass that
    also returns sum(load(r)^2) for the residual history;
  * dots are float64 (K9, deterministic fixed-order reductions);
  * ||s||^2 comes fused out of the back-projection epilogue.

Persistent vectors live in HBM in the chunked layout [chunks][n][f_dev]
that the staged SpMM consumes, so an iteration moves no data to the host
except a handful of scalars.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, engine, matrixstore
from .matrixstore import PRECISIONS

__all__ = ["SolveConfig", "SolveResult", "SolverDivergence", "cgls_solve", "early_stop",
           "residual_curve_report"]


class SolverDivergence(RuntimeError):
    """Raised when an iterate stops being finite (src/solver.py:31-38)."""

    def __init__(self, iteration: int, mode: str, what: str):
        self.iteration = iteration
        self.mode = mode
        super().__init__(f"CGLS diverged at iteration {iteration} in {mode} mode: {what}")


@dataclass(frozen=True)
class SolveConfig:
    """src/solver.py:41-57."""

    max_iters: int = 30
    early_stop_iters: int | None = None
    precision: str = "double"
    seed: int = 0

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.early_stop_iters is not None and not (
                1 <= self.early_stop_iters <= self.max_iters):
            raise ValueError("early_stop_iters must be in [1, max_iters]")
        if self.precision not in PRECISIONS:
            raise ValueError(f"unknown precision {self.precision!r}")


@dataclass
class SolveResult:
    """src/solver.py:60-81."""

    x: np.ndarray = field(repr=False)
    residual_history: list = field(default_factory=list)
    gradient_history: list = field(default_factory=list)
    iteration_seconds: list = field(default_factory=list)
    projections: int = 0
    backprojections: int = 0
    normalization_factors: list = field(default_factory=list)
    mode: str = "double"

    @property
    def iterations(self) -> int:
        return len(self.residual_history)


def early_stop(config: SolveConfig, history: list) -> bool:
    """src/solver.py:120-126."""
    if not history:
        raise ValueError("empty residual history")
    if config.early_stop_iters is None:
        return False
    return len(history) >= config.early_stop_iters


def residual_curve_report(histories: dict) -> str:
    """CSV of relative residuals per mode (src/solver.py:199-223)."""
    if not histories:
        raise ValueError("no residual histories to report")
    modes = sorted(histories)
    for mode, res in histories.items():
        if res.iterations == 0:
            raise ValueError(f"history for mode {mode!r} is empty")
    depth = max(res.iterations for res in histories.values())
    header = ["iteration"]
    for mode in modes:
        header += [f"{mode}_seconds", f"{mode}_rel_residual"]
    lines = [",".join(header)]
    for i in range(depth):
        row = [str(i + 1)]
        for mode in modes:
            res = histories[mode]
            if i < res.iterations:
                row += [f"{sum(res.iteration_seconds[:i + 1]):.6e}",
                        f"{res.residual_history[i]:.9e}"]
            else:
                row += ["", ""]
        lines.append(",".join(row))
    return "\n".join(lines) + "\n"


# measurements and results move between the caller's (rows, slices) layout
# and the device in blocks of rows of about this many bytes
_ROW_BLOCK_BYTES = 512 << 20


class _Vec:
    """A persistent CG vector: payload tensor + dtype code + load factor."""

    __slots__ = ("t", "code", "factor")

    def __init__(self, t, code, factor=1.0):
        self.t, self.code, self.factor = t, code, factor


class LocalComm:
    """Reductions of a single-process solve (identity)."""

    def max_bits(self, t):
        return t

    def sum(self, x: float) -> float:
        return x


class DeviceCG:
    """The device state and kernels of one CGLS solve over one operator.
    ``comm`` supplies the global reductions when the vectors are
    distributed over GPUs (parallel.DomainPartitionedSystem)."""

    def __init__(self, system, n_slices: int, precision: str):
        import torch
        self.sys = system
        self.comm = getattr(system, "comm", None) or LocalComm()
        self.dev = system.device
        self.st = _lib.stream_handle(self.dev)
        self.prec = precision                       # vector-store policy
        self.reduced = precision in ("half", "mixed")
        self.f64 = precision == "double"
        self.code = 0 if self.f64 else 1            # work dtype code
        self.wdt = torch.float64 if self.f64 else torch.float32
        cfg = system.config
        self.op_prec = cfg.precision
        self.F = cfg.ffactor
        self.S = n_slices
        self.n_chunks = -(-n_slices // self.F)
        self.f_dev = system.forward.blocks[0].f_dev
        self.scratch = torch.empty(148 * 8 + 8, dtype=torch.float64, device=self.dev)
        self.scal = torch.zeros(8, dtype=torch.float64, device=self.dev)
        self.bits = torch.zeros(max(self.n_chunks, 1), dtype=torch.int64, device=self.dev)
        sd = {"double": torch.float64, "single": torch.float32}.get(self.op_prec, torch.float16)
        n_max = max(getattr(system, "local_rows", system.num_rows),
                    getattr(system, "local_cols", system.num_cols))
        self.xin_buf = torch.empty(self.n_chunks * n_max * self.f_dev, dtype=sd, device=self.dev)
        self.out_dt = torch.float64 if self.op_prec == "double" else torch.float32
        blks = [b for s in (system.forward, system.adjoint) for b in s.blocks]
        self.part_buf = torch.empty(self.n_chunks * max(b.info.n_cta for b in blks),
                                    dtype=torch.float64, device=self.dev)
        self.events = None           # list -> (is_forward, start, end) per SpMM launch

    # -- helpers ------------------------------------------------------------------
    def numel(self, n):
        return self.n_chunks * n * self.f_dev

    def empty(self, n, dtype=None):
        import torch
        return torch.empty(self.numel(n), dtype=dtype or self.wdt, device=self.dev)

    def sum_sq_to_host(self, t, code, factor=1.0):
        _lib.call("xct_dot", t.data_ptr(), t.data_ptr(), code, t.numel(), float(factor),
                  float(factor), self.scratch.data_ptr(), self.scal.data_ptr(), self.st)
        return self.comm.sum(float(self.scal[0].item()))

    def peak(self, n=1):
        """Global max of the first n max-abs slots (IEEE bits of f64)."""
        self.comm.max_bits(self.bits[:n])
        return self.bits[:n].cpu().numpy().view(np.float64)

    def store(self, v_work, out=None) -> _Vec:
        """_VectorStore.store of a work-dtype vector (src/solver.py:97-103)."""
        import torch
        if not self.reduced:
            return _Vec(v_work, self.code)
        self.bits.zero_()
        _lib.call("xct_maxabs", v_work.data_ptr(), 1, v_work.numel(), 1.0, self.bits.data_ptr(),
                  self.st)
        peak = float(self.peak()[0])
        factor = peak if peak > 0 else 1.0
        if out is None:
            out = torch.empty(v_work.numel(), dtype=torch.float16, device=self.dev)
        _lib.call("xct_axpy", v_work.data_ptr(), 1, 1.0, None, 1, 1.0, 0.0, v_work.numel(),
                  out.data_ptr(), 2, float(np.float32(factor)), None, self.scratch.data_ptr(),
                  None, self.st)
        return _Vec(out, 2, factor)

    def update(self, a: _Vec, b: _Vec, scale: float, out_store=None, want_sumsq=False):
        """out = load(a) + wd(scale) * load(b); stored per the policy.
        Returns (stored _Vec, sum(load(stored)^2) or None, peak)."""
        import torch
        n = a.t.numel()
        fa, fb = float(np.float32(a.factor)), float(np.float32(b.factor))
        if not self.reduced:
            out = out_store if out_store is not None else torch.empty_like(a.t)
            _lib.call("xct_axpy", a.t.data_ptr(), a.code, fa, b.t.data_ptr(), b.code, fb,
                      float(scale), n, out.data_ptr(), self.code, 1.0, None, None, None, self.st)
            ss = self.sum_sq_to_host(out, self.code) if want_sumsq else None
            return _Vec(out, self.code), ss, None
        self.bits.zero_()
        _lib.call("xct_axpy", a.t.data_ptr(), a.code, fa, b.t.data_ptr(), b.code, fb,
                  float(scale), n, None, 2, 1.0, self.bits.data_ptr(), None, None, self.st)
        peak = float(self.peak()[0])
        if not math.isfinite(peak):
            return None, None, peak
        factor = peak if peak > 0 else 1.0
        out = out_store if out_store is not None else torch.empty(n, dtype=torch.float16,
                                                                  device=self.dev)
        _lib.call("xct_axpy", a.t.data_ptr(), a.code, fa, b.t.data_ptr(), b.code, fb,
                  float(scale), n, out.data_ptr(), 2, float(np.float32(factor)), None,
                  self.scratch.data_ptr(), self.scal.data_ptr() if want_sumsq else None,
                  self.st)
        ss = self.comm.sum(float(self.scal[0].item())) if want_sumsq else None
        return _Vec(out, 2, factor), ss, peak

    def apply(self, side, v: _Vec, out):
        """out = op(load(v)) in the chunked layout; returns (factors, ||out||^2)."""
        import torch
        n_in, n_out = side.num_inputs, side.num_outputs
        self.bits.zero_()
        _lib.call("xct_chunk_maxabs_chunked", v.t.data_ptr(), v.code,
                  float(np.float32(v.factor)), n_in, self.n_chunks, self.f_dev,
                  self.bits.data_ptr(), self.st)
        peaks = self.peak(self.n_chunks)
        if not np.all(np.isfinite(peaks)):
            return None, None
        factors = [float(p) if p > 0 else 1.0 for p in peaks]
        fac = torch.tensor(factors, dtype=torch.float64, device=self.dev)
        xin = self.xin_buf[:self.numel(n_in)].view(self.n_chunks, n_in, self.f_dev)
        _lib.call("xct_normalize_chunked", v.t.data_ptr(), v.code, float(np.float32(v.factor)),
                  n_in, self.n_chunks, self.f_dev, fac.data_ptr(), _lib.PREC_CODE[self.op_prec],
                  xin.data_ptr(), self.st)
        if hasattr(side, "exchange_apply"):           # distributed (NCCL) operator
            return factors, self.comm.sum(side.exchange_apply(self, xin, out, fac))
        if len(side.blocks) == 1 and side.input_elements[0] is None:
            blk = side.blocks[0]
            parts = self.part_buf[:self.n_chunks * blk.info.n_cta]
            ev = self.events
            if ev is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            engine.apply_side(blk, xin, out, row_stride=self.f_dev,
                              chunk_stride=n_out * self.f_dev,
                              valid_cols=self.n_chunks * self.f_dev, ffactor_out=self.f_dev,
                              factors=fac, dot_partials=parts, stream=self.st)
            if ev is not None:
                e1.record()
                ev.append((side is self.sys.forward, e0, e1))
            _lib.call("xct_sum_f64", parts.data_ptr(), parts.numel(), self.scal.data_ptr(),
                      self.st)
            return factors, float(self.scal[0].item())
        # data-partitioned operator (one-process emulation): strided path on
        # load(v) in the work dtype, then back to the chunked layout
        loaded = torch.empty((n_in, self.S), dtype=torch.float64, device=self.dev)
        _lib.call("xct_unchunk_f64", v.t.data_ptr(), v.code, float(np.float32(v.factor)), n_in,
                  self.S, self.F, self.f_dev, loaded.data_ptr(), self.st)
        res, _ = self.sys._apply(side, loaded.to(self.wdt))
        tmp = res.to(torch.float64).contiguous()
        oc = 0 if self.out_dt == torch.float64 else 1
        _lib.call("xct_chunk_from_f64", tmp.data_ptr(), n_out, self.S, self.F, self.f_dev, oc,
                  out.data_ptr(), self.st)
        return factors, self.sum_sq_to_host(out, oc)


class CGLSRun:
    """One CGLS solve as explicit steps (used by cgls_solve and bench.py):
    ``start()`` performs the setup and the initial back projection,
    ``step()`` one iteration (1 projection + 1 back projection + updates),
    ``finish()`` returns the SolveResult with x on the host (or device)."""

    def __init__(self, system, y, config: SolveConfig, spmm_events=None):
        import torch
        self.system, self.config = system, config
        self.is_np = not isinstance(y, torch.Tensor)
        yy = np.asarray(y) if self.is_np else y
        self.squeeze = yy.ndim == 1
        n_rows = system.num_rows
        if yy.shape[0] != n_rows:
            raise ValueError(f"measurements have {yy.shape[0]} rays, operator expects {n_rows}")
        self.cg = DeviceCG(system, 1 if self.squeeze else int(yy.shape[1]), config.precision)
        self.cg.events = spmm_events
        self.y = yy
        self.result = SolveResult(x=np.zeros(0), mode=config.precision)
        self.it = 0
        self.done = False

    def start(self) -> bool:
        """Setup and the initial back projection (src/solver.py:141-157).
        Measurements in the caller's row-major layout (host array, pinned or
        not, or a CUDA tensor; float32 or float64) stream through the device
        one block of rows at a time into the chunked work layout (K7
        ``xct_rows_to_chunked``: max|y|, ||y||^2 and wd(y) in one pass), so
        no full float64 copy of y is ever made on the device."""
        import torch
        cg, system = self.cg, self.system
        y = self.y.reshape(system.num_rows, cg.S)
        owned = getattr(system, "row_owned", None)
        n_rows = getattr(system, "local_rows", system.num_rows)
        n_cols = getattr(system, "local_cols", system.num_cols)
        lap = _Lap(cg.dev)
        r = self._store_measurements(y, owned, n_rows)
        lap("start: y upload, norm and store")
        if r is None:
            self.done = True
            self.x = None
            return False
        self.r = r
        if cg.reduced:
            self.x = _Vec(torch.zeros(cg.numel(n_cols), dtype=torch.float16, device=cg.dev), 2, 1.0)
        else:
            self.x = _Vec(torch.zeros(cg.numel(n_cols), dtype=cg.wdt, device=cg.dev), cg.code)
        facs, gamma = cg.apply(system.adjoint, self.r, self.s_buf)
        lap("start: first back projection")
        if facs is None:
            raise SolverDivergence(0, self.config.precision, "residual contains NaN or Inf")
        self.result.backprojections += 1
        self.result.normalization_factors.append(facs)
        s = self._work(self.s_buf)
        self.p = cg.store(s.t) if cg.reduced else _Vec(s.t.clone(), cg.code)
        self.gamma = self.gamma0 = gamma
        return True

    def _store_measurements(self, y, owned, n_rows):
        """r = store(wd(y)), ||y|| and the finite check (src/solver.py:137-150).
        Also allocates the q/s output buffer, which stages wd(y) on the way."""
        import torch
        cg, prec = self.cg, self.config.precision
        S = cg.S
        n_cols = getattr(self.system, "local_cols", self.system.num_cols)
        # one output buffer serves q (projection) and s (back projection): q
        # is dead once r is updated, s is produced after that; before the
        # first back projection it holds wd(y) for the reduced store
        buf = torch.empty(cg.numel(max(n_rows, n_cols)), dtype=cg.out_dt, device=cg.dev)
        self.s_buf = buf[:cg.numel(n_cols)]
        self.q_buf = buf[:cg.numel(n_rows)]
        if cg.reduced:
            work = buf[:cg.numel(n_rows)]
            if cg.out_dt != cg.wdt:
                work = torch.empty(cg.numel(n_rows), dtype=cg.wdt, device=cg.dev)
        else:
            work = torch.empty(cg.numel(n_rows), dtype=cg.wdt, device=cg.dev)
        if S % cg.F or cg.f_dev != cg.F:
            work.zero_()                      # padding slices stay 0
        ybits = torch.zeros(1, dtype=torch.int64, device=cg.dev)
        wbits = torch.zeros(1, dtype=torch.int64, device=cg.dev)
        is_t = isinstance(y, torch.Tensor)
        if owned is not None:                 # distributed: this rank's rays only
            idx = torch.as_tensor(np.asarray(owned, np.int64))
            y = y[idx.to(y.device)] if is_t else np.asarray(y)[np.asarray(owned)]
        if is_t:
            src = y if y.dtype in (torch.float32, torch.float64) else y.to(torch.float64)
            f32_in, on_dev = src.dtype == torch.float32, src.is_cuda
        else:
            src = np.asarray(y)
            if src.dtype not in (np.float32, np.float64):
                src = src.astype(np.float64)
            f32_in, on_dev = src.dtype == np.float32, False
        # blocks of rows: a broadcast (zero-stride) or strided input is only
        # ever materialized one block at a time
        rows_per = max(1, _ROW_BLOCK_BYTES // max(1, S * (4 if f32_in else 8)))
        blocks = [(r0, min(n_rows, r0 + rows_per)) for r0 in range(0, n_rows, rows_per)]
        sums = torch.zeros(max(len(blocks), 1), dtype=torch.float64, device=cg.dev)
        stage = None
        if not on_dev and blocks:
            stage = torch.empty((min(rows_per, n_rows), S),
                                dtype=torch.float32 if f32_in else torch.float64, device=cg.dev)
        for b, (r0, r1) in enumerate(blocks):
            part = src[r0:r1]
            if on_dev:
                blk = part.contiguous()
            else:
                blk = stage[:r1 - r0]
                if isinstance(part, torch.Tensor):
                    blk.copy_(part, non_blocking=part.is_pinned())
                else:
                    _lib.to_device(np.ascontiguousarray(part), blk)
            _lib.call("xct_rows_to_chunked", blk.data_ptr(), 1 if f32_in else 0, r0, r1 - r0,
                      n_rows, S, cg.F, cg.f_dev, cg.code, work.data_ptr(), ybits.data_ptr(),
                      wbits.data_ptr(), cg.scratch.data_ptr(), sums[b:b + 1].data_ptr(), cg.st)
        y_sq = float(sums.cpu().numpy().sum()) if n_rows else 0.0
        cg.comm.max_bits(ybits)
        if not math.isfinite(float(ybits.cpu().numpy().view(np.float64)[0])):
            raise SolverDivergence(0, prec, "measurement data contains NaN or Inf")
        self.y_norm = math.sqrt(cg.comm.sum(y_sq))
        if self.y_norm == 0.0:
            return None
        if not cg.reduced:
            return _Vec(work, cg.code)
        cg.comm.max_bits(wbits)
        peak = float(wbits.cpu().numpy().view(np.float64)[0])
        factor = peak if peak > 0 else 1.0
        r = _Vec(torch.empty(cg.numel(n_rows), dtype=torch.float16, device=cg.dev), 2, factor)
        _lib.call("xct_axpy", work.data_ptr(), cg.code, 1.0, None, cg.code, 1.0, 0.0, work.numel(),
                  r.t.data_ptr(), 2, float(np.float32(factor)), None, cg.scratch.data_ptr(),
                  None, cg.st)
        return r

    def _work(self, buf) -> _Vec:
        cg = self.cg
        return _Vec(buf if cg.out_dt == cg.wdt else buf.to(cg.wdt), cg.code)

    def step(self) -> bool:
        """One iteration (src/solver.py:160-192); False when the solve ends."""
        if self.done or self.it >= self.config.max_iters:
            self.done = True
            return False
        cg, prec, res, system = self.cg, self.config.precision, self.result, self.system
        it = self.it = self.it + 1
        t0 = time.perf_counter()
        if self.gamma == 0.0:
            self.done = True
            return False
        facs, qq = cg.apply(system.forward, self.p, self.q_buf)
        if facs is None:
            raise SolverDivergence(it, prec, "search direction contains NaN or Inf")
        res.projections += 1
        res.normalization_factors.append(facs)
        if qq == 0.0:
            self.done = True
            return False
        alpha = self.gamma / qq
        q = self._work(self.q_buf)
        self.x, _, _ = cg.update(self.x, self.p, alpha, out_store=self.x.t)
        if self.x is None:
            raise SolverDivergence(it, prec, "residual contains NaN or Inf")
        self.r, rr, _ = cg.update(self.r, q, -alpha, out_store=self.r.t, want_sumsq=True)
        if self.r is None or not math.isfinite(rr):
            raise SolverDivergence(it, prec, "residual contains NaN or Inf")
        facs, gamma_new = cg.apply(system.adjoint, self.r, self.s_buf)
        if facs is None:
            raise SolverDivergence(it, prec, "residual contains NaN or Inf")
        res.backprojections += 1
        res.normalization_factors.append(facs)
        if not math.isfinite(gamma_new):
            raise SolverDivergence(it, prec, "gradient norm contains NaN or Inf")
        beta = gamma_new / self.gamma if self.gamma > 0 else 0.0
        self.gamma = gamma_new
        self.p, _, _ = cg.update(self._work(self.s_buf), self.p, beta, out_store=self.p.t)
        if self.p is None:
            raise SolverDivergence(it, prec, "search direction contains NaN or Inf")
        res.residual_history.append(math.sqrt(rr) / self.y_norm)
        res.gradient_history.append(math.sqrt(gamma_new / self.gamma0))
        res.iteration_seconds.append(time.perf_counter() - t0)
        if early_stop(self.config, res.residual_history):
            self.done = True
            return False
        return True

    def finish(self) -> SolveResult:
        import torch
        cg, system = self.cg, self.system
        n_cols, S = getattr(system, "local_cols", system.num_cols), cg.S
        if self.x is None:
            out = np.zeros((n_cols, S))
            if not self.is_np:
                out = torch.zeros((n_cols, S), dtype=torch.float64, device=cg.dev)
        else:
            lap = _Lap(cg.dev)
            fx = float(np.float32(self.x.factor))
            if self.is_np or not self.y.is_cuda:
                # host in -> host out: unchunk one block of rows at a time
                # and copy it through pinned staging into the result (a
                # whole float64 x on the device would cost C*S*8 bytes)
                torch.cuda.synchronize(cg.dev)
                out = _lib.host_array((n_cols, S), np.float64)
                per = max(1, _ROW_BLOCK_BYTES // max(1, S * 8))
                xf = torch.empty((min(per, n_cols), S), dtype=torch.float64, device=cg.dev)
                for r0 in range(0, n_cols, per):
                    r1 = min(n_cols, r0 + per)
                    _lib.call("xct_unchunk_rows_f64", self.x.t.data_ptr(), self.x.code, fx,
                              n_cols, r0, r1 - r0, S, cg.F, cg.f_dev, xf.data_ptr(), cg.st)
                    _lib.to_host(xf[:r1 - r0], out=out[r0:r1])
                if not self.is_np:
                    out = torch.from_numpy(out)
            else:
                out = torch.empty((n_cols, S), dtype=torch.float64, device=cg.dev)
                _lib.call("xct_unchunk_f64", self.x.t.data_ptr(), self.x.code, fx, n_cols, S,
                          cg.F, cg.f_dev, out.data_ptr(), cg.st)
            lap("finish: x to the caller")
        self.result.x = out[:, 0] if self.squeeze else out
        return self.result


class _Lap:
    """Phase timer of the solve's host-facing steps (XCT_VERBOSE only: it
    synchronizes the device)."""

    def __init__(self, dev):
        import os
        self.on = bool(os.environ.get("XCT_VERBOSE"))
        self.dev = dev
        self.t = time.perf_counter()

    def __call__(self, what):
        if not self.on:
            return
        import sys
        import torch
        torch.cuda.synchronize(self.dev)
        now = time.perf_counter()
        print(f"[xct] cgls {what} {now - self.t:.3f} s", file=sys.stderr, flush=True)
        self.t = now


def cgls_solve(system, y, config: SolveConfig) -> SolveResult:
    """Solve min ||y - A x|| by CGLS on the device (src/solver.py:129-196).

    ``y``: (num_rays,) or (num_rays, slices), numpy or a CUDA tensor.
    Returns a SolveResult whose ``x`` is float64 (numpy for numpy input).
    """
    run = CGLSRun(system, y, config)
    if run.start():
        while run.step():
            pass
    return run.finish()
