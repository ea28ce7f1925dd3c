"""Native image-domain partition of the operator over the GPUs of one box
(P_d = world size, src/pipeline.py:84-113).

Rank r owns the voxels T_r of a Hilbert tile segment of the tomogram cut
at EQUAL CUMULATIVE NNZ (hilbert.decompose_weighted; the reference cuts at
equal tile counts, src/hilbert.py:181-200) and the rays G_r of the
reference's sinogram segment (ownership of the ray-side CG vectors).  It
holds two blocks, both built on its own GPU (device Siddon + K4/K5):

  forward  A[:, T_r]    rows = footprint rays F_r ordered by (owner, ray)
  adjoint  A[:, T_r]^T  the same block transposed: rows = T_r, columns = F_r

so both SpMMs cover the same ~nnz/P entries.  Exchanges over NVLink (NCCL
p2p, one message per peer, no gather pass on the K6 side):

  forward  K6 writes element-major partials [F_r][chunk][F]; the rows owned
           by peer q are one contiguous slice, sent in place; the owner sums
           its own partial, then the senders' in ascending rank order (the
           reference's direct plan, src/comm.py:420-472) -- K10
           accumulate_records -- and denormalizes;
  adjoint  the owners of F_r's rays send their normalized inputs (the
           storage dtype: fp16 in mixed mode, half the forward's bytes)
           straight into this rank's element-major K6 input; the output is
           the owned voxels, complete -- no partial-tomogram reduction (the
           reference's sinogram-tile adjoint moves 4.42 C S b_x and is 1.16
           max/mean imbalanced at P_d = 8).

F-chunk waves overlap each wave's exchange with the next wave's K6.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib, engine, hilbert, matrixstore

__all__ = ["NativeDomainBuild", "ForwardSide", "AdjointSide", "exchange_lists"]


def exchange_lists(fp_of: list, seg_of: list, own_rows: np.ndarray, rank: int) -> dict:
    """Index lists of this rank's exchanges (host logic, no device):
    fp_of[s]  footprint rays of rank s, ordered by (owner, ray);
    seg_of[s] [world + 1] offsets of the owner segments of fp_of[s];
    own_rows  this rank's owned rays (sorted).
    Returns positions into own_rows of:
      self_pos   my footprint's own segment (forward accumulate / adjoint gather),
      recv_pos   {s: rays of F_s's segment for me}   (forward accumulate),
      send_idx   {q: rays of F_q's segment for me}   (adjoint gather + send),
    and the segment lengths.  Footprints and ownership must be consistent:
    every ray of an owner segment is owned by that rank (checked)."""
    world = len(fp_of)
    own_rows = np.asarray(own_rows, np.int64)

    def pos_of(rays):
        rays = np.asarray(rays, np.int64)
        p = np.searchsorted(own_rows, rays)
        if len(rays) and (p.max() >= len(own_rows) or not np.array_equal(own_rows[p], rays)):
            raise ValueError("footprint segment holds rays this rank does not own")
        return p.astype(np.int32)

    out = {"self_pos": None, "recv_pos": {}, "send_idx": {}}
    for s in range(world):
        fp, seg = np.asarray(fp_of[s]), np.asarray(seg_of[s])
        if np.any(np.diff(seg) < 0) or seg[-1] != len(fp):
            raise ValueError(f"rank {s}: bad owner segments")
        mine = fp[seg[rank]:seg[rank + 1]]
        if len(mine) > 1 and np.any(np.diff(mine) <= 0):
            raise ValueError(f"rank {s}: footprint segment for rank {rank} is not ascending")
        if s == rank:
            out["self_pos"] = pos_of(mine)
        elif len(mine):
            out["recv_pos"][s] = pos_of(mine)       # forward: s -> me
            out["send_idx"][s] = pos_of(mine)       # adjoint: me -> s (same rays)
    return out


class _Waves:
    WAVES = int(os.environ.get("XCT_EXCHANGE_WAVES", "4"))

    @staticmethod
    def bounds(C):
        W = max(1, min(_Waves.WAVES, C))
        b = [(C * w // W, C * (w + 1) // W) for w in range(W)]
        return [(a, e) for a, e in b if e > a]


class _Stats:
    """Per-application exchange bytes (sent by this rank) and, under
    XCT_EXCHANGE_PROFILE=1, serialized device times of the NCCL phase."""

    def __init__(self):
        self.bytes_out = 0
        self.seconds = 0.0
        self.calls = 0


class IpcBuffer:
    """Device memory this rank allocates and exports over CUDA IPC, and the
    peers' exports mapped here (collective: every rank constructs one)."""

    def __init__(self, nbytes: int, rank: int, world: int):
        import ctypes as C
        import torch.distributed as dist
        L = _lib.lib()
        handle = (C.c_char * 64)()
        ptr = C.c_void_p()
        _lib.check(L.xct_ipc_alloc(max(int(nbytes), 16), C.byref(ptr), handle), "xct_ipc_alloc")
        self.ptr, self.nbytes = int(ptr.value), int(nbytes)
        box = [None] * world
        dist.all_gather_object(box, bytes(handle))
        self.peer = {}
        for q, h in enumerate(box):
            if q == rank:
                self.peer[q] = self.ptr
                continue
            pp = C.c_void_p()
            _lib.check(L.xct_ipc_open(C.create_string_buffer(h, 64), C.byref(pp)), "xct_ipc_open")
            self.peer[q] = int(pp.value)
        self.rank = rank

    def close(self):
        L = _lib.lib()
        for q, pt in self.peer.items():
            if q != self.rank:
                L.xct_ipc_close(pt)
        L.xct_ipc_free(self.ptr)
        self.peer = {}


def fused_default() -> bool:
    """The fused exchange (K6 epilogue stores into peers' buffers) is the
    default; XCT_FUSED_EXCHANGE=0 selects the NCCL p2p waves."""
    return os.environ.get("XCT_FUSED_EXCHANGE", "1") != "0"


class ForwardSide:
    """Projection on this rank: A[:, T_r] -> partials on F_r -> owners.

    Fused exchange (default): K6's epilogue writes each footprint row owned
    by peer q straight into q's receive buffer over NVLink (CUDA IPC
    mapping, element-major [rows][chunks][F]), so the transfer runs tile by
    tile inside the SpMM; a stream-ordered barrier (NCCL all-reduce of one
    word) separates it from the owners' accumulation.  Same bytes, same
    summation order as the NCCL p2p path (bit-identical results)."""

    def __init__(self, block, seg, lists, n_own_rows, rank, world):
        import torch
        dev = block.tensors["values"].device
        self.block, self.blocks = block, [block]
        self.num_inputs, self.num_outputs = block.n_in, n_own_rows
        self.n_fp = block.n_out
        self.seg = [int(v) for v in seg]
        self.rank, self.world = rank, world
        t = lambda a: torch.as_tensor(np.asarray(a, np.int32), device=dev)
        self.self_pos = t(lists["self_pos"])
        self.recv_pos = {s: t(p) for s, p in lists["recv_pos"].items()}
        self.stats = _Stats()
        self.footprints = self.ownership = None         # volume_reports: set by the system
        self.fused = fused_default()
        self._ipc = None
        self._ipc_key = None

    def setup_fused(self, recv_offsets_of):
        """recv_offsets_of[q][s]: first row of sender s's block in rank q's
        receive buffer (all ranks, from an all-gather)."""
        self.recv_off_of = recv_offsets_of

    def _fused_buffers(self, cg, C, fd, eb):
        import torch
        key = (C, fd, eb)
        if self._ipc_key == key:
            return
        if self._ipc is not None:
            self._ipc.close()
        n_recv = sum(int(p.numel()) for p in self.recv_pos.values())
        self._ipc = IpcBuffer(n_recv * C * fd * eb, self.rank, self.world)
        a, b = self.seg[self.rank], self.seg[self.rank + 1]
        self._own = torch.empty((max(b - a, 1), C, fd), dtype=cg.out_dt, device=cg.dev)
        ptrs = []
        for q in range(self.world):
            if q == self.rank:
                ptrs.append(self._own.data_ptr())
            else:
                off = self.recv_off_of[q].get(self.rank, 0)
                ptrs.append(self._ipc.peer[q] + off * C * fd * eb)
        self._ptrs = torch.tensor(ptrs, dtype=torch.int64, device=cg.dev)
        self._seg = torch.tensor(self.seg, dtype=torch.int64, device=cg.dev)
        self._flag = torch.zeros(1, dtype=torch.float32, device=cg.dev)
        self._ipc_key = key

    def _exchange_fused(self, cg, xin, out, fac) -> float:
        import torch
        import torch.distributed as dist
        C, fd = cg.n_chunks, cg.f_dev
        f64 = int(cg.out_dt == torch.float64)
        eb = 8 if f64 else 4
        self._fused_buffers(cg, C, fd, eb)
        o = out.view(C, self.num_outputs, fd)
        dist.all_reduce(self._flag)      # peers are done reading their buffers
        ev = cg.events
        if ev is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        engine.apply_side(self.block, xin, None, row_stride=C * fd, chunk_stride=fd,
                          valid_cols=C * fd, ffactor_out=fd, factors=None, stream=cg.st,
                          out_ptrs=self._ptrs, seg=self._seg)
        if ev is not None:
            e1.record()
            ev.append((True, e0, e1, 1.0))
        for q in range(self.world):
            if q != self.rank:
                self.stats.bytes_out += (self.seg[q + 1] - self.seg[q]) * C * fd * eb
        dist.all_reduce(self._flag)      # every rank's K6 (and its remote stores) done
        o.zero_()
        a, b = self.seg[self.rank], self.seg[self.rank + 1]
        _lib.call("xct_accumulate_records", o.data_ptr(), self.num_outputs, 0,
                  self._own.data_ptr() if b > a else None, self.self_pos.data_ptr(), b - a, C,
                  fd, f64, cg.st)
        off = 0
        for s in sorted(self.recv_pos):
            pos = self.recv_pos[s]
            _lib.call("xct_accumulate_records", o.data_ptr(), self.num_outputs, 0,
                      self._ipc.ptr + off * C * fd * eb, pos.data_ptr(), pos.numel(), C, fd, f64,
                      cg.st)
            off += pos.numel()
        self.stats.calls += 1
        _lib.call("xct_scale_chunks", o.data_ptr(), self.num_outputs * fd, C, fac.data_ptr(), f64,
                  cg.scratch.data_ptr(), cg.scal.data_ptr(), cg.st)
        return float(cg.scal[0].item())

    def exchange_apply(self, cg, xin, out, fac) -> float:
        import torch
        import torch.distributed as dist
        if self.fused and self.world > 1:
            return self._exchange_fused(cg, xin, out, fac)
        C, fd = cg.n_chunks, cg.f_dev
        f64 = int(cg.out_dt == torch.float64)
        eb = 8 if f64 else 4
        o = out.view(C, self.num_outputs, fd)
        prof = os.environ.get("XCT_EXCHANGE_PROFILE") == "1"
        pending = []
        ev = cg.events
        for c0, c1 in _Waves.bounds(C):
            cw = c1 - c0
            part = torch.empty((self.n_fp, cw, fd), dtype=cg.out_dt, device=cg.dev)
            if ev is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            engine.apply_side(self.block, xin[c0:c1], part, row_stride=cw * fd, chunk_stride=fd,
                              valid_cols=cw * fd, ffactor_out=fd, factors=None, stream=cg.st)
            if ev is not None:
                e1.record()
                ev.append((True, e0, e1, cw / C))
            ops, recvs = [], {}
            for q in range(self.world):
                a, b = self.seg[q], self.seg[q + 1]
                if q != self.rank and b > a:
                    ops.append(dist.P2POp(dist.isend, part[a:b], q))
                    self.stats.bytes_out += (b - a) * cw * fd * eb
            for s, pos in self.recv_pos.items():
                recvs[s] = torch.empty((pos.numel(), cw, fd), dtype=cg.out_dt, device=cg.dev)
                ops.append(dist.P2POp(dist.irecv, recvs[s], s))
            if prof:
                torch.cuda.synchronize()
                import time
                t0 = time.perf_counter()
            works = dist.batch_isend_irecv(ops) if ops else []
            if prof:
                for w in works:
                    w.wait()
                torch.cuda.synchronize()
                self.stats.seconds += time.perf_counter() - t0
            pending.append((c0, cw, part, works, recvs))
        for c0, cw, part, works, recvs in pending:
            o[c0:c0 + cw].zero_()
            a, b = self.seg[self.rank], self.seg[self.rank + 1]
            _lib.call("xct_accumulate_records", o.data_ptr(), self.num_outputs, c0,
                      part[a:b].data_ptr() if b > a else None, self.self_pos.data_ptr(), b - a,
                      cw, fd, f64, cg.st)
            for w in works:
                w.wait()                 # the current stream waits for NCCL
            for s in sorted(recvs):
                pos = self.recv_pos[s]
                _lib.call("xct_accumulate_records", o.data_ptr(), self.num_outputs, c0,
                          recvs[s].data_ptr(), pos.data_ptr(), pos.numel(), cw, fd, f64, cg.st)
        self.stats.calls += 1
        _lib.call("xct_scale_chunks", o.data_ptr(), self.num_outputs * fd, C, fac.data_ptr(), f64,
                  cg.scratch.data_ptr(), cg.scal.data_ptr(), cg.st)
        return float(cg.scal[0].item())


class AdjointSide:
    """Back projection on this rank: inputs of F_r gathered from their
    owners, then A[:, T_r]^T -> the owned voxels, complete.  Fused
    (default): the owners' gather kernels store straight into this rank's
    K6 input over NVLink; else NCCL p2p in F-chunk waves."""

    def __init__(self, block, seg, lists, n_own_rows, rank, world):
        import torch
        dev = block.tensors["values"].device
        self.block, self.blocks = block, [block]
        self.num_inputs, self.num_outputs = n_own_rows, block.n_out
        self.n_fp = block.n_in
        self.seg = [int(v) for v in seg]
        self.rank, self.world = rank, world
        t = lambda a: torch.as_tensor(np.asarray(a, np.int32), device=dev)
        self.self_pos = t(lists["self_pos"])
        self.send_idx = {q: t(p) for q, p in lists["send_idx"].items()}
        self.stats = _Stats()
        self.footprints = self.ownership = None
        self.fused = fused_default()
        self._ipc = None
        self._ipc_key = None

    def setup_fused(self, seg_of):
        """seg_of[q]: rank q's owner segments of its footprint (where my
        rays' records go in q's K6 input)."""
        self.seg_of = [[int(v) for v in sg] for sg in seg_of]

    def _exchange_fused(self, cg, xin, out, fac) -> float:
        """Owners push their normalized inputs straight into the consumers'
        K6 input buffers over NVLink: one gather kernel per consumer whose
        destination is the consumer's buffer (CUDA IPC mapping) -- gather
        and transfer in one pass, no NCCL staging.  In F-chunk waves: the
        receive buffer is wave-major ([wave][footprint][chunks of the wave]
        [record]), wave w+1's gathers run on a side stream while K6 consumes
        wave w, a flag all-reduce per wave marks its stores landed."""
        import torch
        import torch.distributed as dist
        C, fd = cg.n_chunks, cg.f_dev
        eb = xin.element_size()
        rec = fd * eb
        key = (C, fd, eb)
        if self._ipc_key != key:
            if self._ipc is not None:
                self._ipc.close()
            self._ipc = IpcBuffer(self.n_fp * C * rec, self.rank, self.world)
            self._flag = torch.zeros(1, dtype=torch.float32, device=cg.dev)
            self._side = torch.cuda.Stream(device=cg.dev)
            self._ipc_key = key
        o = out.view(C, self.num_outputs, fd)
        blk = self.block
        n_cta = blk.info.n_cta
        parts = torch.empty(C * n_cta, dtype=torch.float64, device=cg.dev)
        prof = os.environ.get("XCT_EXCHANGE_PROFILE") == "1"
        waves = _Waves.bounds(C) if not prof else [(0, C)]
        main = torch.cuda.current_stream(cg.dev)
        side = self._side
        dist.all_reduce(self._flag)           # consumers are done with their inputs
        if prof:
            import time
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        side.wait_stream(main)
        st_side = int(side.cuda_stream)
        ready = []
        a, b = self.seg[self.rank], self.seg[self.rank + 1]
        with torch.cuda.stream(side):
            for c0, c1 in waves:
                cw = c1 - c0
                base = self.n_fp * c0 * rec              # this wave's region, my buffer
                _lib.call("xct_gather_records", xin.data_ptr(), self.num_inputs,
                          self.self_pos.data_ptr(), b - a, c0, cw, rec,
                          self._ipc.ptr + base + a * cw * rec if b > a else None, st_side)
                for q, idx in self.send_idx.items():
                    n_fp_q = self.seg_of[q][-1]
                    dst = self._ipc.peer[q] + n_fp_q * c0 * rec + \
                        self.seg_of[q][self.rank] * cw * rec
                    _lib.call("xct_gather_records", xin.data_ptr(), self.num_inputs,
                              idx.data_ptr(), idx.numel(), c0, cw, rec, dst, st_side)
                    self.stats.bytes_out += idx.numel() * cw * rec
                dist.all_reduce(self._flag)       # every producer's wave stores landed
                e = torch.cuda.Event()
                e.record(side)
                ready.append(e)
        if prof:
            torch.cuda.synchronize()
            self.stats.seconds += time.perf_counter() - t0
        ev = cg.events
        for (c0, c1), e in zip(waves, ready):
            cw = c1 - c0
            main.wait_event(e)
            if ev is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            engine.apply_side_ptr(blk, self._ipc.ptr + self.n_fp * c0 * rec, cw, o[c0:c1],
                                  row_stride=fd, chunk_stride=self.num_outputs * fd,
                                  valid_cols=cw * fd, ffactor_out=fd, factors=fac[c0:c1],
                                  dot_partials=parts[c0 * n_cta:c1 * n_cta], stream=cg.st,
                                  x_chunk_stride=1, x_elem_stride=cw)
            if ev is not None:
                e1.record()
                ev.append((False, e0, e1, cw / C))
        self.stats.calls += 1
        _lib.call("xct_sum_f64", parts.data_ptr(), parts.numel(), cg.scal.data_ptr(), cg.st)
        return float(cg.scal[0].item())

    def exchange_apply(self, cg, xin, out, fac) -> float:
        import torch
        import torch.distributed as dist
        if self.fused and self.world > 1:
            return self._exchange_fused(cg, xin, out, fac)
        C, fd = cg.n_chunks, cg.f_dev
        rec = fd * xin.element_size()
        o = out.view(C, self.num_outputs, fd)
        prof = os.environ.get("XCT_EXCHANGE_PROFILE") == "1"
        waves = _Waves.bounds(C)
        ev = cg.events
        blk = self.block
        parts = torch.empty(C * blk.info.n_cta, dtype=torch.float64, device=cg.dev)

        def issue(c0, c1):
            cw = c1 - c0
            xfp = torch.empty((self.n_fp, cw, fd), dtype=xin.dtype, device=cg.dev)
            a, b = self.seg[self.rank], self.seg[self.rank + 1]
            _lib.call("xct_gather_records", xin.data_ptr(), self.num_inputs,
                      self.self_pos.data_ptr(), b - a, c0, cw, rec,
                      xfp[a:b].data_ptr() if b > a else None, cg.st)
            ops, bufs = [], []
            for q, idx in self.send_idx.items():
                buf = torch.empty((idx.numel(), cw, fd), dtype=xin.dtype, device=cg.dev)
                _lib.call("xct_gather_records", xin.data_ptr(), self.num_inputs, idx.data_ptr(),
                          idx.numel(), c0, cw, rec, buf.data_ptr(), cg.st)
                ops.append(dist.P2POp(dist.isend, buf, q))
                bufs.append(buf)
                self.stats.bytes_out += idx.numel() * cw * rec
            for s in range(self.world):
                a, b = self.seg[s], self.seg[s + 1]
                if s != self.rank and b > a:
                    ops.append(dist.P2POp(dist.irecv, xfp[a:b], s))
            if prof:
                torch.cuda.synchronize()
                import time
                t0 = time.perf_counter()
            works = dist.batch_isend_irecv(ops) if ops else []
            if prof:
                for w in works:
                    w.wait()
                torch.cuda.synchronize()
                self.stats.seconds += time.perf_counter() - t0
            return xfp, works, bufs

        nxt = issue(*waves[0])
        for i, (c0, c1) in enumerate(waves):
            xfp, works, bufs = nxt
            if i + 1 < len(waves):
                nxt = issue(*waves[i + 1])          # next wave's exchange in flight
            for w in works:
                w.wait()
            cw = c1 - c0
            if ev is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            engine.apply_side(blk, xfp, o[c0:c1], row_stride=fd,
                              chunk_stride=self.num_outputs * fd, valid_cols=cw * fd,
                              ffactor_out=fd, factors=fac[c0:c1],
                              dot_partials=parts[c0 * blk.info.n_cta:c1 * blk.info.n_cta],
                              stream=cg.st, x_chunk_stride=1, x_elem_stride=cw)
            if ev is not None:
                e1.record()
                ev.append((False, e0, e1, cw / C))
            del bufs
        self.stats.calls += 1
        _lib.call("xct_sum_f64", parts.data_ptr(), parts.numel(), cg.scal.data_ptr(), cg.st)
        return float(cg.scal[0].item())


class NativeDomainBuild:
    """Per-rank device build of the two blocks (see the module docstring)."""

    BAND_NNZ = 2.5e9

    def __init__(self, geometry, config, rank, world, dev):
        from . import pipeline
        self.g, self.cfg, self.rank, self.world, self.dev = geometry, config, rank, world, dev
        self.sa = pipeline.StreamedAssembly(geometry, config)
        self.G = pipeline._side_group(config, "forward")
        self.G_a = pipeline._side_group(config, "adjoint")
        self.rw = pipeline._rows_per_warp(config, kind="forward")
        self.rw_a = pipeline._rows_per_warp(config, kind="adjoint")
        self.st = _lib.stream_handle(dev)

    def _part(self, d_ip, d_ix, d_v, n_rows, n_cols, plan, B, nk):
        """Device K5 of one part; grouped rows (FP32 default G = 4) or a
        declined device build go through the host builder (global column
        ids, the plan's own key tables) and are uploaded."""
        cfg, exp = self.cfg, self.exp
        if matrixstore.device_build_supported(plan, cfg.precision):
            try:
                return matrixstore.build_format_device(d_ip, d_ix, d_v, n_rows, n_cols, plan,
                                                       cfg.precision, cfg.ffactor, exp,
                                                       cfg.smem_budget_effective,
                                                       cfg.order == "native", B, nk, self.dev)
            except matrixstore.DeviceBuildUnsupported:
                pass
        hf = matrixstore.build_format(_lib.to_host(d_ip), _lib.to_host(d_ix[:int(d_ip[-1])]),
                                      _lib.to_host(d_v[:int(d_ip[-1])]), n_rows, n_cols, plan,
                                      cfg.precision, cfg.ffactor, exp, cfg.smem_budget_effective,
                                      schedule=cfg.order == "native")
        return matrixstore.host_part(hf, cfg.precision, cfg.ffactor, n_cols, n_rows, exp, self.dev)

    def _filter(self, ip, ix, v, rows, cmap):
        """Device CSR restricted to the columns with cmap >= 0 (rewritten to
        cmap), row structure kept; returns (counts, indptr, indices, values)."""
        import torch
        cnt = torch.empty(rows, dtype=torch.int64, device=self.dev)
        _lib.call("xct_csr_filter_map", ip.data_ptr(), ix.data_ptr(), v.data_ptr(), rows, None,
                  cmap.data_ptr(), cnt.data_ptr(), None, None, None, self.st)
        optr = torch.zeros(rows + 1, dtype=torch.int64, device=self.dev)
        torch.cumsum(cnt, 0, out=optr[1:])
        m = int(optr[-1])
        oi = torch.empty(max(m, 1), dtype=torch.int32, device=self.dev)
        ov = torch.empty(max(m, 1), dtype=torch.float64, device=self.dev)
        _lib.call("xct_csr_filter_map", ip.data_ptr(), ix.data_ptr(), v.data_ptr(), rows, None,
                  cmap.data_ptr(), None, optr.data_ptr(), oi.data_ptr(), ov.data_ptr(), self.st)
        return cnt, optr, oi, ov

    def run(self):
        import torch
        from . import pipeline
        g, cfg, dev, rank, world = self.g, self.cfg, self.dev, self.rank, self.world
        n, R, Cn = g.grid_n, g.num_rays, g.num_voxels
        sa = self.sa
        G, rw = self.G, self.rw
        ta = matrixstore.forward_tile_height(n, rw, cfg.warps_per_cta, G, g.num_angles)
        chunks = sa._chunks(ta)
        exp = sa._exponent(chunks) if cfg.precision in ("half", "mixed") else 0
        self.exp = exp
        # pass 1: entries per voxel -> tomogram cut at equal cumulative nnz
        counts = torch.zeros(Cn, dtype=torch.int64, device=dev)
        for k0, k1 in chunks:
            ip, ix, _ = sa._siddon(k0, k1)
            _lib.call("xct_csr_col_counts", ip.data_ptr(), ix.data_ptr(), (k1 - k0) * n, 0, Cn,
                      counts.data_ptr(), self.st)
            del ip, ix
        h_counts = counts.cpu().numpy()
        tomo = hilbert.decompose_weighted(hilbert.TileGrid("tomogram", n, n, cfg.tile_size),
                                          world, h_counts)
        sino = hilbert.decompose(hilbert.TileGrid("sinogram", g.num_angles,
                                                  g.num_detector_cols, cfg.tile_size), world)
        self.tomo, self.sino = tomo, sino
        cols = tomo[rank].elements
        owner_of_ray = np.empty(R, np.int32)
        for q, s in enumerate(sino):
            owner_of_ray[s.elements] = q
        cm_g = np.full(Cn, -1, np.int32)
        cm_g[cols] = cols.astype(np.int32)
        cm_l = np.full(Cn, -1, np.int32)
        cm_l[cols] = np.arange(len(cols), dtype=np.int32)
        d_cmg, d_cml = torch.from_numpy(cm_g).to(dev), torch.from_numpy(cm_l).to(dev)
        # pass 2: forward block A[:, T_r], per view chunk
        parts, fps, base = [], [], 0
        for k0, k1 in chunks:
            rows = (k1 - k0) * n
            ip, ix, v = sa._siddon(k0, k1)
            cnt, optr, oi, ov = self._filter(ip, ix, v, rows, d_cmg)
            del ip, ix, v
            keep = torch.nonzero(cnt).reshape(-1)
            if keep.numel() == 0:
                continue
            bip = torch.cat((optr[keep], optr[-1:])).contiguous()
            keep_h = keep.cpu().numpy()
            plan = matrixstore.assign_forward_regimes(
                matrixstore.forward_plan(g.num_angles, n, rw, cfg.warps_per_cta, k0, k1,
                                         row_group=G), g.angles, n)
            pos = np.full(rows, -1, np.int64)
            pos[keep_h] = np.arange(len(keep_h))
            cr = plan.cta_rows
            cr = np.where(cr >= 0, pos[np.maximum(cr - k0 * n, 0)], -1)
            live = (cr >= 0).any(axis=1)
            plan.cta_rows, plan.cta_table = cr[live].astype(np.int32), plan.cta_table[live]
            part = self._part(bip, oi, ov, len(keep_h), Cn, plan, n, n)
            gm = part.tensors["group_map"]
            part.tensors["group_map"] = d_cml[gm.long()]
            part.fp_base = base
            parts.append(part)
            fps.append(k0 * n + keep_h)
            base += len(keep_h)
            del oi, ov, optr, cnt, bip
        fp_all = np.concatenate(fps) if fps else np.empty(0, np.int64)
        order = np.argsort(owner_of_ray[fp_all], kind="stable")
        fp_sorted = fp_all[order]
        final_pos = np.empty(len(fp_all), np.int64)
        final_pos[order] = np.arange(len(fp_all))
        d_final = torch.from_numpy(final_pos.astype(np.int32)).to(dev)
        for part in parts:
            cr = part.tensors["cta_rows"]
            part.tensors["cta_rows"] = torch.where(cr >= 0, d_final[(cr.long() + part.fp_base)
                                                                    .clamp_min(0)], cr)
        seg = np.searchsorted(owner_of_ray[fp_sorted], np.arange(world + 1)).astype(np.int64)
        fwd = matrixstore.combine_device_parts(parts, cfg.precision, cfg.ffactor, len(cols),
                                               len(fp_sorted), exp, dev)
        # pass 3: adjoint block A[:, T_r]^T, bands of the owned voxels
        ray2pos = np.full(R, -1, np.int32)
        ray2pos[fp_sorted] = np.arange(len(fp_sorted), dtype=np.int32)
        d_ray2pos = torch.from_numpy(ray2pos).to(dev)
        c_local = counts[torch.from_numpy(cols).to(dev)]
        tz = matrixstore.adjoint_tile_height(n, self.rw_a, cfg.warps_per_cta, self.G_a)
        row_nnz = np.zeros(n, np.int64)
        np.add.at(row_nnz, cols // n, h_counts[cols])
        bands, z0 = [], 0
        while z0 < n:
            z1, acc = z0, 0
            while z1 < n and (z1 == z0 or acc + row_nnz[z1:z1 + tz].sum() <= self.BAND_NNZ):
                acc += row_nnz[z1:z1 + tz].sum()
                z1 = min(n, z1 + tz)
            bands.append((z0, z1))
            z0 = z1
        aparts = []
        for z0, z1 in bands:
            lo, hi = (int(np.searchsorted(cols, z0 * n)), int(np.searchsorted(cols, z1 * n)))
            if hi <= lo:
                continue
            nb = hi - lo
            t_ip = torch.zeros(nb + 1, dtype=torch.int64, device=dev)
            torch.cumsum(c_local[lo:hi], 0, out=t_ip[1:])
            m = int(t_ip[-1])
            t_rows = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
            t_vals = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
            cur = torch.zeros(nb, dtype=torch.int32, device=dev)
            prev = torch.zeros(nb, dtype=torch.int32, device=dev)
            for k0, k1 in chunks:
                rows = (k1 - k0) * n
                ip, ix, v = sa._siddon(k0, k1)
                _, optr, oi, ov = self._filter(ip, ix, v, rows, d_cml)
                del ip, ix, v
                _lib.call("xct_csr_transpose_band", optr.data_ptr(), oi.data_ptr(), ov.data_ptr(),
                          rows, k0 * n, 32 * n, lo, hi, t_ip.data_ptr(), cur.data_ptr(),
                          prev.data_ptr(), t_rows.data_ptr(), t_vals.data_ptr(), self.st)
                del optr, oi, ov
            plan = matrixstore.adjoint_plan(g.num_angles, n, self.rw_a, cfg.warps_per_cta, z0, z1,
                                            row_group=self.G_a)
            cr = plan.cta_rows
            cr = np.where(cr >= 0, cm_l[np.maximum(cr, 0)], -1)
            cr = np.where(cr >= 0, cr - lo, -1)
            live = (cr >= 0).any(axis=1)
            plan.cta_rows, plan.cta_table = cr[live].astype(np.int32), plan.cta_table[live]
            part = self._part(t_ip, t_rows, t_vals, nb, R, plan, g.num_detector_cols,
                              g.num_angles)
            gm = part.tensors["group_map"]
            part.tensors["group_map"] = d_ray2pos[gm.long()]
            cr = part.tensors["cta_rows"]
            part.tensors["cta_rows"] = torch.where(cr >= 0, cr + lo, cr)
            aparts.append(part)
            del t_ip, t_rows, t_vals, cur, prev
        adj = matrixstore.combine_device_parts(aparts, cfg.precision, cfg.ffactor, len(fp_sorted),
                                               len(cols), exp, dev)
        self.nnz_local = int(fwd.info.nnz)
        return fwd, adj, fp_sorted, seg, cols
