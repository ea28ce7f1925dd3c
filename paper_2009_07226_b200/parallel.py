"""Multi-GPU plumbing: one process per GPU, torch.distributed over NCCL.

Slice-batch parallelism (P_b, src/cli.py:158-200): the slices are split
into contiguous groups (first S mod P_b groups get one more) and every GPU
runs an independent CGLS on its group with its own alpha/beta -- no
data-path collective.  Every GPU needs the whole operator; it is built once
on the source rank and broadcast over NVLink (NCCL) instead of being rebuilt
per rank, so host memory and build time do not scale with the GPU count.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import matrixstore, pipeline  # noqa: F401

__all__ = ["slice_groups", "broadcast_system", "MatrixInfo", "DomainPartitionedSystem",
           "NcclComm"]


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
    meta = [None]
    if rank == src:
        if len(system.forward.blocks) != 1 or system.forward.input_elements[0] is not None:
            # every rank must learn of the error, or the others block in the
            # broadcast below
            meta = [{"error": "broadcast_system supports the single-block (P_d = 1) operator"}]
        else:
            m = system.matrix
            meta = [dict(num_rows=int(m.num_rows), num_cols=int(m.num_cols), nnz=int(m.nnz),
                         num_angles=int(getattr(m, "num_angles", m.num_rows)),
                         num_detector_cols=int(getattr(m, "num_detector_cols", 1)),
                         exp=int(system.value_scale_exp))]
    dist.broadcast_object_list(meta, src=src, device=dev)
    meta = meta[0]
    if "error" in meta:
        raise ValueError(meta["error"])
    fwd = _bcast_side(system.forward.blocks[0] if rank == src else None, src, rank, dev)
    adj = _bcast_side(system.adjoint.blocks[0] if rank == src else None, src, rank, dev)
    if rank == src:
        return system
    info = MatrixInfo(meta["num_rows"], meta["num_cols"], meta["nnz"], meta["num_angles"],
                      meta["num_detector_cols"])
    return pipeline.AssembledSystem.from_sides(info, config, geometry, fwd, adj, meta["exp"])


# ---------------------------------------------------------------------------
# Data-partitioned operator over GPUs (P_d = world size)
# ---------------------------------------------------------------------------

class NcclComm:
    """Global reductions of a distributed CGLS (NCCL over NVLink)."""

    def __init__(self, dev):
        import torch
        self.dev = dev
        self._s = torch.zeros(1, dtype=torch.float64, device=dev)

    def max_bits(self, t):
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)     # max of non-negative f64 bits
        return t

    def sum(self, x: float) -> float:
        import torch.distributed as dist
        self._s.fill_(x)
        dist.all_reduce(self._s)
        return float(self._s.item())


class _ExchangeProfile:
    """XCT_EXCHANGE_PROFILE=1: per-phase device times of one partitioned
    application (phases serialized; a diagnosis aid, not a timing mode)."""

    def __init__(self, rank):
        import os
        self.on = os.environ.get("XCT_EXCHANGE_PROFILE") == "1"
        self.rank, self.laps = rank, []
        if self.on:
            import time
            import torch
            torch.cuda.synchronize()
            self.t = time.perf_counter()

    def lap(self, what):
        if not self.on:
            return
        import time
        import torch
        torch.cuda.synchronize()
        now = time.perf_counter()
        self.laps.append((what, now - self.t))
        self.t = now

    def report(self, side):
        if self.on and self.rank == 0:
            import sys
            print(f"[xct] exchange {side}: " +
                  ", ".join(f"{w} {t * 1e3:.1f} ms" for w, t in self.laps), file=sys.stderr)


class _DistSide:
    """One direction of the partitioned operator on this rank: the local
    staged block (rows = footprint elements) and the exchange that turns its
    partial products into the owned outputs (K10 + NCCL p2p)."""

    def __init__(self, block, fp_ids, own_ids, in_ids, fp_of, own_of, rank, dev):
        import torch
        self.block = block
        self.blocks = [block]
        self.num_inputs, self.num_outputs = len(in_ids), len(own_ids)
        self.n_fp = len(fp_ids)
        self.rank, self.peers = rank, len(fp_of)
        self.footprints, self.ownership = fp_of, own_of   # all ranks' (volume_reports)
        t = lambda a: torch.as_tensor(np.asarray(a, np.int32), device=dev)
        # send and receive sides pair rows by position in ascending element
        # order: every footprint and ownership list must be strictly ascending
        for name, arr in [("footprint", fp_ids), ("ownership", own_ids)] + \
                [(f"footprint of rank {s}", f) for s, f in enumerate(fp_of)] + \
                [(f"ownership of rank {s}", o) for s, o in enumerate(own_of)]:
            a = np.asarray(arr)
            if len(a) > 1 and not np.all(np.diff(a) > 0):
                raise ValueError(f"{name} is not strictly ascending")
        owner = {}
        # positions of each peer's owned elements inside my footprint (send)
        self.send = {}
        for q, own_q in enumerate(own_of):
            pos = np.nonzero(np.isin(fp_ids, own_q, assume_unique=True))[0]
            if q == rank:
                self.self_src = t(pos)
                self.self_dst = t(np.searchsorted(own_ids, fp_ids[pos]))
            elif len(pos):
                self.send[q] = t(pos)
        # where each peer's contributions land in my owned outputs (recv)
        self.recv = {}
        for s, fp_s in enumerate(fp_of):
            if s == rank:
                continue
            hit = np.intersect1d(fp_s, own_ids, assume_unique=True)
            if len(hit):
                self.recv[s] = t(np.searchsorted(own_ids, hit))
        del owner

    # F-chunk waves per application: the exchange of wave w (gather, NCCL
    # p2p over NVLink) runs on NCCL's stream while K6 computes wave w + 1
    import os as _os
    WAVES = int(_os.environ.get("XCT_EXCHANGE_WAVES", "4"))

    def exchange_apply(self, cg, xin, out, fac) -> float:
        """Local partial SpMM, exchange, reduction in the reference's direct
        plan order (owner first, then senders ascending), denormalize.
        The F-chunks go in waves so each wave's exchange overlaps the next
        wave's SpMM; every output element still sums the same partials in
        the same order.  Returns the local sum of squares of the owned
        outputs."""
        import torch
        import torch.distributed as dist
        from . import _lib, engine
        C, fd = cg.n_chunks, cg.f_dev
        f64 = int(cg.out_dt == torch.float64)
        partial = torch.empty((C, self.n_fp, fd), dtype=cg.out_dt, device=cg.dev)
        o = out.view(C, self.num_outputs, fd)
        W = max(1, min(self.WAVES, C))
        bounds = [(C * w // W, C * (w + 1) // W) for w in range(W)]
        bounds = [(a, b) for a, b in bounds if b > a]
        ev = cg.events

        def gather(idx, c0, c1):
            buf = torch.empty((c1 - c0, idx.numel(), fd), dtype=cg.out_dt, device=cg.dev)
            _lib.call("xct_gather_rows", partial[c0:c1].data_ptr(), self.n_fp, idx.data_ptr(),
                      idx.numel(), c1 - c0, fd, f64, buf.data_ptr(), cg.st)
            return buf

        prof = _ExchangeProfile(self.rank)
        if prof.on:
            bounds = [(0, C)]         # phases serialized and timed (diagnosis only)
        pending = []
        for c0, c1 in bounds:
            if ev is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            engine.apply_side(self.block, xin[c0:c1], partial[c0:c1], row_stride=fd,
                              chunk_stride=self.n_fp * fd, valid_cols=(c1 - c0) * fd,
                              ffactor_out=fd, factors=None, stream=cg.st)
            if ev is not None:
                e1.record()
                ev.append((self is cg.sys.forward, e0, e1, (c1 - c0) / C))
            prof.lap("K6")
            sends = {q: gather(idx, c0, c1) for q, idx in self.send.items()}
            prof.lap("gather")
            recvs = {s: torch.empty((c1 - c0, idx.numel(), fd), dtype=cg.out_dt,
                                    device=cg.dev)
                     for s, idx in self.recv.items()}
            ops = [dist.P2POp(dist.isend, b, q) for q, b in sends.items()]
            ops += [dist.P2POp(dist.irecv, b, s) for s, b in recvs.items()]
            works = dist.batch_isend_irecv(ops) if ops else []
            if prof.on:
                for r in works:
                    r.wait()
            prof.lap(f"nccl p2p {sum(b.numel() * b.element_size() for b in sends.values()) / 1e9:.2f} GB out")
            pending.append((c0, c1, works, sends, recvs))
        for c0, c1, works, sends, recvs in pending:
            ow = o[c0:c1]
            ow.zero_()
            own = gather(self.self_src, c0, c1)
            _lib.call("xct_accumulate_rows", ow.data_ptr(), self.num_outputs, own.data_ptr(),
                      self.self_dst.data_ptr(), self.self_dst.numel(), c1 - c0, fd, f64, cg.st)
            for r in works:
                r.wait()            # the current stream waits for NCCL; the host does not
            for s in sorted(recvs):
                _lib.call("xct_accumulate_rows", ow.data_ptr(), self.num_outputs,
                          recvs[s].data_ptr(), self.recv[s].data_ptr(), self.recv[s].numel(),
                          c1 - c0, fd, f64, cg.st)
        prof.lap("accumulate")
        _lib.call("xct_scale_chunks", o.data_ptr(), self.num_outputs * fd, C, fac.data_ptr(), f64,
                  cg.scratch.data_ptr(), cg.scal.data_ptr(), cg.st)
        prof.lap("scale")
        prof.report("forward" if self is cg.sys.forward else "adjoint")
        return float(cg.scal[0].item())


class DomainPartitionedSystem:
    """Operator partitioned over the GPUs by Hilbert tile segments of both
    planes (src/pipeline.py:104-113, src/hilbert.py:181-200): rank r owns
    voxels T_r and rays G_r, holds A[:, T_r] (footprint rays) and
    A[G_r, :]^T (footprint voxels), and exchanges partial sinograms /
    tomograms with its peers over NVLink (NCCL p2p) once per application.
    Duck-types the AssembledSystem surface used by solver.CGLSRun; the CGLS
    vectors are distributed (each rank holds its owned elements)."""

    def __init__(self, geometry, config, src: int = 0):
        import torch
        import torch.distributed as dist
        from . import geometry as geo
        from . import pipeline
        from .pipeline import column_block, hilbert_subdomains, row_block_transposed
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.comm = NcclComm(self.device)
        self.config, self.geometry = config, geometry
        g = geometry
        self.num_rows, self.num_cols = g.num_rays, g.num_voxels
        if config.order != "reference" and os.environ.get("XCT_DOMAIN_LEGACY") != "1":
            self._init_native(g, config)
            pipeline.configure_execution((self.forward, self.adjoint), config)
            return
        tomo, sino = hilbert_subdomains(g, config.tile_size, self.world)
        self.col_owned = tomo[self.rank].elements
        self.row_owned = sino[self.rank].elements
        self.local_cols, self.local_rows = len(self.col_owned), len(self.row_owned)
        rw = pipeline._rows_per_warp(config)
        schedule = config.order == "native"
        metas = None
        if config.order != "reference" and (
                config.build == "streamed" or
                (config.build == "auto" and 1.2 * g.num_angles * g.grid_n ** 2 > 4e9)):
            self._init_streamed(g, config, tomo, sino)
            pipeline.configure_execution((self.forward, self.adjoint), config)
            return
        err = None
        if self.rank == src:
            try:
                built, metas, exp = self._build_all(g, config, tomo, sino, rw, schedule)
            except Exception as e:            # reported to every rank below
                err = f"{type(e).__name__}: {e}"
        box = [{"error": err} if err else metas]
        dist.broadcast_object_list(box, src=src, device=self.device)
        if isinstance(box[0], dict) and box[0].get("error"):
            raise RuntimeError(f"domain build on rank {src} failed: {box[0]['error']}")
        metas = box[0]
        self._finish_legacy(g, config, tomo, sino, src, built if self.rank == src else None, metas)

    def _build_all(self, g, config, tomo, sino, rw, schedule):
        """Rank src: every rank's blocks from the whole matrix (legacy path,
        reference order)."""
        from . import geometry as geo
        from .pipeline import column_block, row_block_transposed
        if True:
            A = geo.build_system_matrix(g)
            ip, ix, v = A.host_csr32()
            exp = (matrixstore.half_rescale_exponent(v)
                   if config.precision in ("half", "mixed") else 0)
            R, Cn = g.num_rays, g.num_voxels
            n = g.grid_n
            built = []
            if config.order != "reference":
                # the single-GPU tiles (sinogram / voxel tiles, band keys),
                # restricted to each rank's block
                gf = matrixstore.assign_forward_regimes(
                    matrixstore.forward_plan(g.num_angles, n,
                                             pipeline._rows_per_warp(config, kind="forward"),
                                             config.warps_per_cta,
                                             row_group=pipeline._side_group(config, "forward")),
                    g.angles, n)
                ga = matrixstore.adjoint_plan(g.num_angles, n,
                                              pipeline._rows_per_warp(config, kind="adjoint"),
                                              config.warps_per_cta,
                                              row_group=pipeline._side_group(config, "adjoint"))
            for q in range(self.world):
                cols, rays = tomo[q].elements, sino[q].elements
                bip, bix, bv, f_fp = column_block(ip, ix, v, R, Cn, cols)
                t_ip, t_ix, t_v, a_fp = row_block_transposed(ip, ix, v, rays)
                sides = []
                for (pip, pix, pv, nr, nc, rows_g, cols_g, gplan) in (
                        (bip, bix, bv, len(f_fp), len(cols), f_fp, cols,
                         gf if config.order != "reference" else None),
                        (t_ip, t_ix, t_v, len(a_fp), len(rays), a_fp, rays,
                         ga if config.order != "reference" else None)):
                    if config.order == "reference":
                        plan = matrixstore.reference_plan(
                            pip, pix, nr, nc, config.block_partitions,
                            config.stage_capacity_bytes, config.ffactor, config.precision, rw,
                            config.warps_per_cta)
                        budget = pipeline.smem_budget_for(config, plan)
                    else:
                        plan = matrixstore.restrict_plan(gplan, rows_g, cols_g)
                        budget = config.smem_budget_effective
                    sides.append(matrixstore.build_format(pip, pix, pv, nr, nc, plan,
                                                          config.precision, config.ffactor,
                                                          exp, budget, schedule))
                built.append((sides, f_fp, a_fp))
            geo.clear_matrix_cache()
            del A, ip, ix, v
            metas = [dict(exp=exp, f_fp=b[1], a_fp=b[2]) for b in built]
        return built, metas, exp

    def _finish_legacy(self, g, config, tomo, sino, src, built, metas):
        import torch
        from . import pipeline
        self.value_scale_exp = metas[0]["exp"]
        fp_fwd = [m["f_fp"] for m in metas]
        fp_adj = [m["a_fp"] for m in metas]
        # ship every rank its two formats (uploaded by the source, NCCL p2p)
        mine = []
        for k, (n_in, n_out) in enumerate(((len(self.col_owned), len(fp_fwd[self.rank])),
                                           (len(self.row_owned), len(fp_adj[self.rank])))):
            side = None
            for q in range(self.world):
                if self.rank == src:
                    hf = built[q][0][k]
                    ins = (len(tomo[q].elements), len(sino[q].elements))[k]
                    outs = (len(fp_fwd[q]), len(fp_adj[q]))[k]
                    blk = matrixstore.upload_format(hf, config.precision, config.ffactor, ins,
                                                    outs, self.value_scale_exp, self.device)
                    if q == src:
                        side = blk
                    else:
                        _send_side(blk, q)
                    del blk
                elif q == self.rank:
                    side = _recv_side(src, self.device)
            mine.append(side)
        if self.rank == src:
            del built
        torch.cuda.empty_cache()
        self.forward = _DistSide(mine[0], fp_fwd[self.rank], self.row_owned, self.col_owned,
                                 fp_fwd, [s.elements for s in sino], self.rank, self.device)
        self.adjoint = _DistSide(mine[1], fp_adj[self.rank], self.col_owned, self.row_owned,
                                 fp_adj, [s.elements for s in tomo], self.rank, self.device)
        pipeline.configure_execution((self.forward, self.adjoint), config)

    def _init_native(self, g, config):
        """Native partition (domain.py): equal-nnz tomogram cut, per-rank
        device build of A[:, T_r] and its transpose, owner-ordered
        footprints, no gather on the K6 side of either exchange."""
        import torch.distributed as dist
        from . import domain
        if config.precision not in ("single", "mixed", "half", "double"):
            raise ValueError(f"unknown precision {config.precision!r}")
        b = domain.NativeDomainBuild(g, config, self.rank, self.world, self.device)
        fwd, adj, fp, seg, cols = b.run()
        self.value_scale_exp = b.exp
        self.tomogram_subdomains, self.sinogram_subdomains = b.tomo, b.sino
        self.col_owned = cols
        self.row_owned = b.sino[self.rank].elements
        self.local_cols, self.local_rows = len(self.col_owned), len(self.row_owned)
        box = [None] * self.world
        dist.all_gather_object(box, (fp, seg))
        fp_of, seg_of = [x[0] for x in box], [x[1] for x in box]
        lists = domain.exchange_lists(fp_of, seg_of, self.row_owned, self.rank)
        self.forward = domain.ForwardSide(fwd, seg, lists, self.local_rows, self.rank, self.world)
        # receive layout of the fused exchange: senders' blocks in ascending
        # sender order, each rank's offsets known to all
        offs, at = {}, 0
        for s_ in sorted(lists["recv_pos"]):
            offs[s_] = at
            at += len(lists["recv_pos"][s_])
        box2 = [None] * self.world
        dist.all_gather_object(box2, offs)
        self.forward.setup_fused(box2)
        self.adjoint = domain.AdjointSide(adj, seg, lists, self.local_rows, self.rank, self.world)
        self.adjoint.setup_fused(seg_of)
        own_rays = [s.elements for s in b.sino]
        self.forward.footprints, self.forward.ownership = fp_of, own_rays
        self.adjoint.footprints, self.adjoint.ownership = fp_of, own_rays
        self.native = True
        dist.barrier()

    def exchange_stats(self) -> dict:
        """Bytes this rank sent per application (and, under
        XCT_EXCHANGE_PROFILE=1, the serialized NCCL time) for each side."""
        out = {}
        for name, side in (("projection", self.forward), ("backprojection", self.adjoint)):
            st = getattr(side, "stats", None)
            if st is None or not st.calls:
                continue
            out[name] = {"bytes_out_per_application": st.bytes_out / st.calls,
                         "nccl_seconds_per_application": st.seconds / st.calls,
                         "applications": st.calls}
        return out

    def _init_streamed(self, g, config, tomo, sino):
        """Every rank builds its own blocks (no whole matrix anywhere)."""
        import os
        import torch
        import torch.distributed as dist
        fparts, f_fp, aparts, a_fp, exp = build_rank_blocks_streamed(
            g, config, tomo, sino, self.rank, self.device)
        self.value_scale_exp = exp
        box = [None] * self.world
        dist.all_gather_object(box, (f_fp, a_fp))
        fp_fwd = [b[0] for b in box]
        fp_adj = [b[1] for b in box]
        fwd = matrixstore.upload_format(fparts, config.precision, config.ffactor,
                                        len(self.col_owned), len(f_fp), exp, self.device)
        adj = matrixstore.upload_format(aparts, config.precision, config.ffactor,
                                        len(self.row_owned), len(a_fp), exp, self.device)
        del fparts, aparts
        torch.cuda.empty_cache()
        self.forward = _DistSide(fwd, f_fp, self.row_owned, self.col_owned, fp_fwd,
                                 [s.elements for s in sino], self.rank, self.device)
        self.adjoint = _DistSide(adj, a_fp, self.col_owned, self.row_owned, fp_adj,
                                 [s.elements for s in tomo], self.rank, self.device)
        dist.barrier()

    def hbm_bytes(self) -> int:
        return self.forward.block.hbm_bytes() + self.adjoint.block.hbm_bytes()

    def volume_reports(self) -> dict:
        """Per-level byte accounting of this partition's exchange, the
        reference's `VolumeReport` per side (src/pipeline.py:192-194) with
        P_d = world size, planned over ``config.topology`` (comm.py).  Every
        rank holds all footprints, so no collective is needed."""
        from . import comm
        cfg = self.config
        topo = cfg.topology if cfg.topology is not None else comm.default_topology()
        placement = comm.map_partitions(1, self.world, topo)
        planner = (comm.plan_hierarchical if cfg.comm_strategy == "hierarchical"
                   else comm.plan_direct)
        eb = matrixstore.element_bytes(cfg.precision)
        return {name: planner(dict(enumerate(side.footprints)),
                              dict(enumerate(side.ownership)), placement,
                              ffactor=cfg.ffactor, elem_bytes=eb)[1]
                for name, side in (("projection", self.forward),
                                   ("backprojection", self.adjoint))}

    def gather_x(self, x_local):
        """Assemble the full (num_cols, S) estimate on every rank (small
        problems / tests)."""
        import torch.distributed as dist
        parts = [None] * self.world
        dist.all_gather_object(parts, (self.col_owned, np.asarray(x_local)))
        full = np.zeros((self.num_cols,) + np.asarray(x_local).shape[1:])
        for cols, xl in parts:
            full[cols] = xl
        return full


def _send_side(side, dst):
    import torch.distributed as dist
    dist.send_object_list([matrixstore.side_meta(side)], dst=dst,
                          device=side.tensors["values"].device)
    for k in sorted(side.tensors):
        dist.send(side.tensors[k].view(-1).view(__import__("torch").uint8), dst=dst)


def _recv_side(src, dev):
    import torch
    import torch.distributed as dist
    box = [None]
    dist.recv_object_list(box, src=src, device=dev)
    meta = box[0]
    tensors = {}
    for k in sorted(meta["tensors"]):
        shape, dtype = meta["tensors"][k]
        t = torch.empty(shape, dtype=getattr(torch, dtype), device=dev)
        dist.recv(t.view(-1).view(torch.uint8), src=src)
        tensors[k] = t
    return matrixstore.side_from_meta(meta, tensors)


def _filter_map(ip, ix, v, rows, row_keep, col_map, st, dev):
    """Device CSR restriction (xct_csr_filter_map) -> host (counts, idx, val)."""
    import torch
    from . import _lib
    cnt = torch.empty(rows, dtype=torch.int64, device=dev)
    rk = row_keep.data_ptr() if row_keep is not None else None
    _lib.call("xct_csr_filter_map", ip.data_ptr(), ix.data_ptr(), v.data_ptr(), rows, rk,
              col_map.data_ptr(), cnt.data_ptr(), None, None, None, st)
    optr = torch.zeros(rows + 1, dtype=torch.int64, device=dev)
    torch.cumsum(cnt, 0, out=optr[1:])
    m = int(optr[-1])
    oi = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    ov = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
    _lib.call("xct_csr_filter_map", ip.data_ptr(), ix.data_ptr(), v.data_ptr(), rows, rk,
              col_map.data_ptr(), None, optr.data_ptr(), oi.data_ptr(), ov.data_ptr(), st)
    return cnt.cpu().numpy(), oi[:m].cpu().numpy(), ov[:m].cpu().numpy()


def build_rank_blocks_streamed(g, config, tomo, sino, rank, dev, n_threads=None):
    """This rank's forward block A[:, T_r] and back-projection block
    A[G_r, :]^T built without the whole matrix: Siddon regenerated per view
    chunk on this GPU, restricted on the device (xct_csr_filter_map), staged
    per chunk / voxel band on the host.  Every rank builds its own blocks in
    parallel.  Returns (fwd parts, fwd footprint rays, adj parts, adj
    footprint voxels, value_scale_exp)."""
    import torch
    from . import _lib, pipeline
    sa = pipeline.StreamedAssembly(g, config)
    rw = sa.rw
    n, R, Cn = g.grid_n, g.num_rays, g.num_voxels
    st = _lib.stream_handle(dev)
    Gf, Ga, rw_a = (pipeline._side_group(config, "forward"), pipeline._side_group(config, "adjoint"),
                    sa.rw_a)
    ta = matrixstore.forward_tile_height(n, rw, config.warps_per_cta, Gf, g.num_angles)
    chunks = sa._chunks(ta)
    exp = sa._exponent(chunks) if config.precision in ("half", "mixed") else 0
    schedule = config.order == "native"
    cols, rays = tomo[rank].elements, sino[rank].elements
    # forward: columns -> local owned index, rows = rays touching them
    cmap = np.full(Cn, -1, np.int32)
    cmap[cols] = np.arange(len(cols), dtype=np.int32)
    d_cmap = torch.from_numpy(cmap).to(dev)
    fparts, fps = [], []
    base = 0
    for k0, k1 in chunks:
        ip, ix, v = sa._siddon(k0, k1)
        rows = (k1 - k0) * n
        cnt, bix, bv = _filter_map(ip, ix, v, rows, None, d_cmap, st, dev)
        keep = np.nonzero(cnt)[0]
        fp = (k0 * n + keep).astype(np.int64)
        if len(fp) == 0:
            continue
        bip = np.concatenate(([0], np.cumsum(cnt[keep]))).astype(np.int64)
        gplan = matrixstore.assign_forward_regimes(
            matrixstore.forward_plan(g.num_angles, n, rw, config.warps_per_cta, k0, k1,
                                     row_group=Gf),
            g.angles, n)
        plan = matrixstore.restrict_plan(gplan, fp, cols)
        hf = matrixstore.build_format(bip, bix, bv, len(fp), len(cols), plan, config.precision,
                                      config.ffactor, exp, config.smem_budget_effective, schedule)
        hf.cta_rows = np.where(hf.cta_rows >= 0, hf.cta_rows + base, -1).astype(np.int32)
        fparts.append(hf)
        fps.append(fp)
        base += len(fp)
    f_fp = np.concatenate(fps) if fps else np.empty(0, np.int64)
    # back projection: owned rays x voxel bands, transposed per band
    rkeep = np.zeros(R, np.uint8)
    rkeep[rays] = 1
    d_rkeep = torch.from_numpy(rkeep).to(dev)
    tz = matrixstore.adjoint_tile_height(n, rw_a, config.warps_per_cta, Ga)
    per = max(1, int(sa.BAND_NNZ // (1.2 * g.num_angles * n)))
    per = max(tz, per // tz * tz)
    aparts, aps = [], []
    base = 0
    for z0 in range(0, n, per):
        z1 = min(n, z0 + per)
        lo, hi = z0 * n, z1 * n
        bmap = np.full(Cn, -1, np.int32)
        bmap[lo:hi] = np.arange(hi - lo, dtype=np.int32)
        d_bmap = torch.from_numpy(bmap).to(dev)
        counts, idx, val = [], [], []
        for k0, k1 in chunks:
            ip, ix, v = sa._siddon(k0, k1)
            rows = (k1 - k0) * n
            cnt, bix, bv = _filter_map(ip, ix, v, rows, d_rkeep[k0 * n:k1 * n], d_bmap, st, dev)
            keep_rows = rkeep[k0 * n:k1 * n].astype(bool)
            counts.append(cnt[keep_rows])            # owned rays, ascending
            idx.append(bix)
            val.append(bv)
        bip = np.zeros(len(rays) + 1, np.int64)
        np.cumsum(np.concatenate(counts), out=bip[1:])
        bix, bv = np.concatenate(idx), np.concatenate(val)
        t_ip, t_ix, t_v = pipeline._transpose(bip, bix, bv, len(rays), hi - lo)
        nz = np.nonzero(np.diff(t_ip))[0]                   # band voxels touched
        if len(nz) == 0:
            continue
        vp = (lo + nz).astype(np.int64)
        sub_ip = np.concatenate((t_ip[nz], t_ip[-1:])).astype(np.int64)   # drop empty rows
        gplan = matrixstore.adjoint_plan(g.num_angles, n, rw_a, config.warps_per_cta, z0, z1,
                                         row_group=Ga)
        plan = matrixstore.restrict_plan(gplan, vp, rays)
        hf = matrixstore.build_format(sub_ip, t_ix, t_v, len(vp), len(rays), plan,
                                      config.precision, config.ffactor, exp,
                                      config.smem_budget_effective, schedule)
        hf.cta_rows = np.where(hf.cta_rows >= 0, hf.cta_rows + base, -1).astype(np.int32)
        aparts.append(hf)
        aps.append(vp)
        base += len(vp)
    a_fp = np.concatenate(aps) if aps else np.empty(0, np.int64)
    return fparts, f_fp, aparts, a_fp, exp
