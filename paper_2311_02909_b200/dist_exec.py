"""B200 executor of the distributed samplers: one process per GPU.

Replicated mode (cfg4, dist.py:417-429): rank r samples the contiguous batch
range of group r with the fused device bulk sampler; no communication.

1.5D partitioned mode (cfg5, Alg. 2, dist.py:308-378) for GraphSAGE:
the grid is p/c rows x c columns (rank = i*c + j); A is split into p/c
contiguous vertex-range block rows, block i held by the c ranks of grid row
i; the batches are split into p/c groups, group i sampled by grid row i.
Per layer, rank (i, j):

  1. row fetch — sparsity aware: for stage q < p/c^2 it asks the owner of
     block k = j*stages + q, rank (k, j), for exactly the distinct frontier
     vertices of its group that fall in block k (NnzCols), and receives those
     A rows (degrees are global metadata, so the reply is just the packed
     column ids).  P2P send/recv inside the grid column (NCCL over NVLink).
  2. sample-then-reduce — every frontier row is one-hot, so its P row lives
     entirely in one block: rank (i, j) samples exactly the rows whose vertex
     lies in its column's vertex range [V_j, V_{j+1}) from the fetched rows
     (gb_sage_layer_sample), writing picks at their global frontier
     positions; an all-reduce (sum) of the frontier inside grid row i
     assembles the complete frontier.  This replaces the reference's P
     all-reduce (37-66x larger) by s ids per row.
  3. extraction on the complete frontier (gb_sage_layer_extract), identical
     on the c replicas.

The result of grid row i equals the serial bulk of group i (same global
row keys), so the concatenation over grid rows equals the serial epoch.
"""

from __future__ import annotations

import ctypes
import os
import sys
import time

import numpy as np

from . import _lib
from .dist import ProcessGrid, _bounds
from .errors import ContractViolation
from .sampler import LayerSample, SampledEpoch, SamplerKind


def _torch():
    import torch

    return torch


def _staged():
    """gloo process group: device tensors travel through host copies (the
    single-GPU multi-process parity test and the CPU host-logic tests)."""
    import torch.distributed as dist

    return dist.get_backend() == "gloo"


def _all_reduce(t, op=None, group=None):
    import torch.distributed as dist

    op = dist.ReduceOp.SUM if op is None else op
    if _staged() and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


def _all_gather(parts, t, group=None):
    import torch.distributed as dist

    if _staged() and t.is_cuda:
        hp = [p.cpu() for p in parts]
        dist.all_gather(hp, t.cpu(), group=group)
        for p, h in zip(parts, hp):
            p.copy_(h)
    else:
        dist.all_gather(parts, t, group=group)


def _all_gather_into(out, t):
    import torch.distributed as dist

    if _staged():
        parts = list(out.view(-1, t.numel()).unbind(0))
        _all_gather(parts, t)
    else:
        dist.all_gather_into_tensor(out, t)


# bytes this process handed to the transport (payload of the executor's
# messages, size exchanges excluded): the ledger's words describe exactly
# this traffic (tests/dist_exec_check.py)
WIRE = {"bytes": 0}


def exchange(sends, recv_sizes, group_ranks, dtype, device, count_wire=True):
    """Point-to-point exchange inside a group: sends {peer: tensor},
    recv_sizes {peer: count}; returns {peer: tensor}.  Grouped isend/irecv
    (NCCL over NVLink on GPUs; gloo through host copies for the single-GPU
    multi-process and CPU tests)."""
    import torch.distributed as dist

    torch = _torch()
    staged = _staged()
    wire = torch.device("cpu") if staged else device
    ops, out = [], {}
    me = dist.get_rank()
    for peer, n in recv_sizes.items():
        if peer == me:
            continue
        buf = torch.empty(int(n), dtype=dtype, device=wire)
        out[peer] = buf
        if n:
            ops.append(dist.P2POp(dist.irecv, buf, peer))
    for peer, t in sends.items():
        if peer == me:
            out[peer] = t
            continue
        if t.numel():
            ops.append(dist.P2POp(dist.isend, t.contiguous().to(wire), peer))
            if count_wire:
                WIRE["bytes"] += t.numel() * t.element_size()
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if staged:
        out = {p: (t if p == me else t.to(device)) for p, t in out.items()}
    return out


def exchange_counts(sends, group_ranks, device):
    """Every member learns how many elements each peer sends it."""
    import torch.distributed as dist

    torch = _torch()
    me = dist.get_rank()
    cnt_out = {p: torch.tensor([int(sends.get(p, torch.empty(0)).numel())], dtype=torch.int64,
                               device=device) for p in group_ranks}
    got = exchange(cnt_out, {p: 1 for p in group_ranks}, group_ranks, torch.int64, device,
                   count_wire=False)
    return {p: int(got[p].item()) if p != me else int(cnt_out[me].item()) for p in group_ranks}


class BlockGraph:
    """This rank's share of a 1.5D-partitioned graph (partition_block_rows,
    dist.py:200-214): the block row of its grid row — rows [lo, hi) of A as
    a CSR with global column ids — plus the global degree metadata the
    sampler needs (degrees all-gathered once over the process group, the
    global row offsets scanned from them, the per-degree replay tables built
    from them).  No other block's columns are resident on this GPU.

    `tables` is a DeviceGraph whose rowptr is the global one and whose
    column array is a stub: every column read of the 1.5D samplers goes to
    a block CSR (local, fetched or a peer's).
    """

    def __init__(self, n, grid: ProcessGrid, row0, brp, bcol, nnz):
        import torch.distributed as dist

        from .sparse import DeviceGraph

        torch = _torch()
        self.n, self.grid = int(n), grid
        self.row0, self.brp, self.nnz = int(row0), brp, int(nnz)
        self.bcol = bcol  # padded by GB_COL_PAD (16-B streaming loads)
        bounds = _bounds(self.n, grid.rows)
        sizes = np.diff(bounds)
        maxb = int(sizes.max())
        dev = brp.device
        mine = torch.zeros(maxb, dtype=torch.int32, device=dev)
        mine[: brp.numel() - 1] = (brp[1:] - brp[:-1]).to(torch.int32)
        allb = torch.empty(grid.p * maxb, dtype=torch.int32, device=dev)
        _all_gather_into(allb, mine)
        allb = allb.view(grid.p, maxb)
        self.gdeg = torch.cat([allb[grid.rank(i, 0), : int(sizes[i])] for i in range(grid.rows)])
        rowptr = torch.zeros(self.n + 1, dtype=torch.int64, device=dev)
        torch.cumsum(self.gdeg.long(), 0, out=rowptr[1:])
        stub = torch.zeros(_lib.GB_COL_PAD, dtype=torch.int32, device=dev)
        self.tables = DeviceGraph(self.n, rowptr, stub, int(rowptr[-1].item()))

    @classmethod
    def rmat(cls, n, m, symmetric, grid: ProcessGrid, seed=0):
        """Block row of the synthetic R-MAT graph (gb_rmat_block): only the
        block is built on this GPU."""
        import torch.distributed as dist

        from .graphgen import rmat_device_block

        i, _ = grid.coords(dist.get_rank())
        bounds = _bounds(int(n), grid.rows)
        lo, hi = int(bounds[i]), int(bounds[i + 1])
        brp, bcol, nnz = rmat_device_block(n, m, symmetric, lo, hi, seed=seed)
        return cls(n, grid, lo, brp, bcol, nnz)

    @classmethod
    def from_full(cls, full, grid: ProcessGrid):
        """Cut this rank's block out of a replicated DeviceGraph (tests)."""
        import torch.distributed as dist

        torch = _torch()
        i, _ = grid.coords(dist.get_rank())
        bounds = _bounds(full.n, grid.rows)
        lo, hi = int(bounds[i]), int(bounds[i + 1])
        a0, a1 = int(full.rowptr[lo].item()), int(full.rowptr[hi].item())
        brp = (full.rowptr[lo:hi + 1] - a0).contiguous()
        bcol = torch.zeros(a1 - a0 + _lib.GB_COL_PAD, dtype=torch.int32, device=brp.device)
        bcol[: a1 - a0] = full.col[a0:a1]
        return cls(full.n, grid, lo, brp, bcol, a1 - a0)

    def resident_bytes(self):
        """Graph bytes held on this GPU: block CSR + global degree metadata."""
        return int(self.brp.numel() * 8 + self.bcol.numel() * 4 + self.gdeg.numel() * 4 +
                   self.tables.rowptr.numel() * 8)


class Sage15D:
    """1.5D partitioned GraphSAGE bulk sampler over real processes.

    part: this rank's BlockGraph (only its grid row's block resident), or a
    replicated DeviceGraph from which the block is cut (tests).
    """

    def __init__(self, part, grid: ProcessGrid, fanouts, batch_size, mode="pfree",
                 ledger=None, fetch="rows"):
        import torch.distributed as dist

        torch = _torch()
        if not dist.is_initialized() or dist.get_world_size() != grid.p:
            raise ContractViolation("Sage15D needs torch.distributed with world_size == grid.p")
        if not isinstance(part, BlockGraph):
            part = BlockGraph.from_full(part, grid)
        self.part = part
        self.grid, self.fanouts, self.b = grid, tuple(int(s) for s in fanouts), int(batch_size)
        self.mode, self.ledger = mode, ledger
        if fetch not in ("rows", "owner", "p2p", "split"):
            raise ContractViolation(f"unknown fetch mode {fetch!r}")
        # "rows": Alg. 2 row fetch; "owner": owner samples, returns picks;
        # "p2p": owner reads requests from and writes picks into peer memory;
        # "split": the grid row's replicas split its batches and run the
        # single-GPU dedup bulk on rows read from the owners' memory
        self.fetch = fetch
        self._p2p = None
        self.rank = dist.get_rank()
        self.i, self.j = grid.coords(self.rank)
        self.n = part.n
        self.tables = part.tables  # global rowptr + replay tables, no columns
        self.gdeg = part.gdeg
        self.bounds = _bounds(self.n, grid.rows)
        self.row0 = part.row0
        self.brp = part.brp
        self.bcol = part.bcol[: part.nnz]
        st = grid.stages
        self.V0 = int(self.bounds[self.j * st])
        self.V1 = int(self.bounds[(self.j + 1) * st])
        self.row_groups = [dist.new_group(grid.row_group(r)) for r in range(grid.rows)]
        self.col_ranks = grid.col_group(self.j)
        self.row_ranks = grid.row_group(self.i)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.stats = {"fetch_ids": 0, "fetch_words": 0, "reduce_words": 0}
        # per-phase wall time (ms, host clock around device-synchronised
        # phases) when profile is set: the α–β cost-model check
        self.profile = False
        self.phase_ms = {"fetch": 0.0, "reduce": 0.0}

    def _phase(self, name, t0):
        import time

        torch = _torch()
        if not self.profile:
            return time.perf_counter()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if name:
            self.phase_ms[name] += 1e3 * (t1 - t0)
        return t1

    # -- step 1: sparsity-aware row fetch ------------------------------------------
    def _peer_block(self):
        """This rank's block CSR in symmetric memory (padded to the largest
        block of any rank), so requesters read rows straight out of it."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        torch = _torch()
        if getattr(self, "_pblk", None) is not None:
            return self._pblk
        sz = torch.tensor([self.brp.numel(), self.bcol.numel()], dtype=torch.int64,
                          device=self.dev)
        _all_reduce(sz, op=dist.ReduceOp.MAX)
        nr, nc = (int(x) for x in sz.tolist())
        grp = dist.group.WORLD.group_name
        rp = symm_mem.empty(max(nr, 1), dtype=torch.int64, device=self.dev)
        cl = symm_mem.empty(max(nc, 1) + _lib.GB_COL_PAD, dtype=torch.int32, device=self.dev)
        rp[: self.brp.numel()].copy_(self.brp)
        cl[: self.bcol.numel()].copy_(self.bcol)
        cl[self.bcol.numel():].zero_()
        # the block lives only in symmetric memory from here on
        nb, nc = self.brp.numel(), self.bcol.numel()
        self.brp, self.bcol = rp[:nb], cl[:nc]
        self.part.brp, self.part.bcol = rp[:nb], cl
        self._pblk = {"rp": rp, "rp_h": symm_mem.rendezvous(rp, grp), "cl": cl,
                      "cl_h": symm_mem.rendezvous(cl, grp)}
        self._pblk["rp_h"].barrier(channel=0)
        return self._pblk

    def fetch_rows_p2p(self, U):
        """fetch_rows with the messages replaced by peer reads: the A rows of
        U are gathered straight from each block owner's CSR in symmetric
        memory (gb_gather_rows on the peer pointers).  Same local CSR."""
        torch = _torch()
        L = _lib.lib()
        pb = self._peer_block()
        grid, st = self.grid, self.grid.stages
        d = self.gdeg[U.long()].long()
        lrowptr = torch.zeros(U.numel() + 1, dtype=torch.int64, device=self.dev)
        lrowptr[1:] = torch.cumsum(d, 0)
        nnz = int(lrowptr[-1].item())
        lcol = torch.zeros(nnz + _lib.GB_COL_PAD, dtype=torch.int32, device=self.dev)
        for q in range(st):
            kblk = self.j * st + q
            owner = grid.rank(kblk, self.j)
            lo, hi = int(self.bounds[kblk]), int(self.bounds[kblk + 1])
            sel = torch.nonzero((U >= lo) & (U < hi)).flatten()
            if sel.numel() == 0:
                continue
            ids = U[sel].to(torch.int32).contiguous()
            offs = lrowptr[sel].contiguous()
            _lib.check(L.gb_gather_rows(ids.numel(), _lib.ptr(ids), lo,
                                        ctypes.c_void_p(pb["rp_h"].buffer_ptrs[owner]),
                                        ctypes.c_void_p(pb["cl_h"].buffer_ptrs[owner]),
                                        _lib.ptr(offs), _lib.ptr(lcol), _lib.stream_ptr()),
                       "gb_gather_rows")
            if owner != self.rank:
                self.stats["fetch_ids"] += ids.numel()
        if prof:
            ev[1].record()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            if self.rank == 0:
                print(f"GB_PROF15 fetch: prep {1e3 * (t1 - t0):.3f} ms, gathers "
                      f"{1e3 * (t2 - t1):.3f} ms wall / {ev[0].elapsed_time(ev[1]):.3f} ms device, "
                      f"rows {U.numel()}, entries {nnz}", file=sys.stderr)
        return lrowptr, lcol

    def fetch_rows_any(self, U):
        """A rows of any sorted distinct vertices U from their block owners'
        memory (grid row b, this rank's column: every replica of a grid row
        holds its block), as a local CSR — peer reads, no messages."""
        torch = _torch()
        L = _lib.lib()
        pb = self._peer_block()
        prof = os.environ.get("GB_PROF15") == "1"
        if prof:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        d = self.gdeg[U.long()].long()
        lrowptr = torch.zeros(U.numel() + 1, dtype=torch.int64, device=self.dev)
        lrowptr[1:] = torch.cumsum(d, 0)
        nnz = int(lrowptr[-1].item())
        lcol = torch.zeros(nnz + _lib.GB_COL_PAD, dtype=torch.int32, device=self.dev)
        if prof:
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
        for b in range(self.grid.rows):
            owner = self.grid.rank(b, self.j)
            lo, hi = int(self.bounds[b]), int(self.bounds[b + 1])
            sel = torch.nonzero((U >= lo) & (U < hi)).flatten()
            if sel.numel() == 0:
                continue
            ids = U[sel].to(torch.int32).contiguous()
            offs = lrowptr[sel].contiguous()
            _lib.check(L.gb_gather_rows(ids.numel(), _lib.ptr(ids), lo,
                                        ctypes.c_void_p(pb["rp_h"].buffer_ptrs[owner]),
                                        ctypes.c_void_p(pb["cl_h"].buffer_ptrs[owner]),
                                        _lib.ptr(offs), _lib.ptr(lcol), _lib.stream_ptr()),
                       "gb_gather_rows")
            if owner != self.rank:
                self.stats["fetch_ids"] += ids.numel()
        if prof:
            ev[1].record()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            if self.rank == 0:
                print(f"GB_PROF15 fetch: prep {1e3 * (t1 - t0):.3f} ms, gathers "
                      f"{1e3 * (t2 - t1):.3f} ms wall / {ev[0].elapsed_time(ev[1]):.3f} ms device, "
                      f"rows {U.numel()}, entries {nnz}", file=sys.stderr)
        return lrowptr, lcol

    def fetch_rows(self, U):
        """A rows of the sorted distinct vertices U (all in this column's
        range) as a local CSR (rowptr over U, cols)."""
        torch = _torch()
        if self.fetch == "p2p":
            return self.fetch_rows_p2p(U)
        grid, st, L = self.grid, self.grid.stages, _lib.lib()
        replies = []
        for q in range(st):
            kblk = self.j * st + q
            owner = grid.rank(kblk, self.j)
            lo, hi = int(self.bounds[kblk]), int(self.bounds[kblk + 1])
            ids = U[(U >= lo) & (U < hi)].contiguous()
            sends = {owner: ids}
            counts = exchange_counts(sends, self.col_ranks, self.dev)
            reqs = exchange(sends, {p: counts[p] for p in self.col_ranks if self.rank == owner or
                                    p == self.rank}, self.col_ranks, torch.int32, self.dev)
            # owner: serve every request of this stage from the local block
            out = {}
            if self.rank == owner:
                for p in self.col_ranks:
                    rid = reqs.get(p)
                    if rid is None or rid.numel() == 0:
                        continue
                    d = self.gdeg[rid.long()].long()
                    off = torch.zeros(rid.numel() + 1, dtype=torch.int64, device=self.dev)
                    off[1:] = torch.cumsum(d, 0)
                    buf = torch.empty(max(int(off[-1].item()), 1), dtype=torch.int32,
                                      device=self.dev)
                    _lib.check(L.gb_gather_rows(rid.numel(), _lib.ptr(rid), self.row0,
                                                _lib.ptr(self.brp), _lib.ptr(self.bcol),
                                                _lib.ptr(off), _lib.ptr(buf), _lib.stream_ptr()),
                               "gb_gather_rows")
                    out[p] = buf[: int(off[-1].item())]
                    if self.ledger is not None and p != self.rank and out[p].numel():
                        self.ledger.charge(self.rank, "row-data", 1, out[p].numel())
            if self.ledger is not None and owner != self.rank and ids.numel():
                self.ledger.charge(self.rank, "gather-cols", 1, ids.numel())
            want = int(self.gdeg[ids.long()].long().sum().item()) if ids.numel() else 0
            self.stats["fetch_ids"] += ids.numel() if owner != self.rank else 0
            self.stats["fetch_words"] += want if owner != self.rank else 0
            got = exchange(out, {owner: want}, self.col_ranks, torch.int32, self.dev)
            replies.append(got.get(owner, torch.empty(0, dtype=torch.int32, device=self.dev))
                           if want else torch.empty(0, dtype=torch.int32, device=self.dev))
        d = self.gdeg[U.long()].long()
        lrowptr = torch.zeros(U.numel() + 1, dtype=torch.int64, device=self.dev)
        lrowptr[1:] = torch.cumsum(d, 0)
        nnz = int(lrowptr[-1].item())
        lcol = torch.zeros(nnz + _lib.GB_COL_PAD, dtype=torch.int32, device=self.dev)
        if nnz:
            lcol[:nnz] = torch.cat(replies)
        return lrowptr, lcol

    # -- step 1+2, owner-computes variant ------------------------------------------------
    def owner_sample(self, rv, mine, deg, fptr, brow, k, stride, batch_offset, s, seed, epoch,
                     depth, fcol):
        """Ship (vertex, global row key) of every row in block k to its owner,
        which samples it from its local A rows with the same keyed replay
        (gb_sage_sample_keyed) and returns only the sorted picks."""
        torch = _torch()
        L = _lib.lib()
        grid, st, dev = self.grid, self.grid.stages, self.dev
        R = rv.numel()
        ridx = torch.arange(R, device=dev)
        b = torch.searchsorted(brow, ridx, right=True) - 1
        keys = (batch_offset + b) * stride + (ridx - brow[b])
        take_all = torch.minimum(deg.long(), torch.full_like(deg, s).long())
        for q in range(st):
            kblk = self.j * st + q
            owner = grid.rank(kblk, self.j)
            lo, hi = int(self.bounds[kblk]), int(self.bounds[kblk + 1])
            sel = torch.nonzero(mine & (rv >= lo) & (rv < hi) & (deg > 0)).flatten()
            req = torch.stack([rv[sel].long(), keys[sel]], 1).flatten().contiguous()
            counts = exchange_counts({owner: req}, self.col_ranks, dev)
            reqs = exchange({owner: req}, {p: counts[p] for p in self.col_ranks
                                           if self.rank == owner or p == self.rank},
                            self.col_ranks, torch.int64, dev)
            replies = {}
            if self.rank == owner:
                for p in self.col_ranks:
                    r = reqs.get(p)
                    if r is None or r.numel() == 0:
                        continue
                    r = r.view(-1, 2)
                    v = r[:, 0]
                    d = self.gdeg[v].contiguous()
                    tk = torch.minimum(d.long(), torch.full_like(d, s).long())
                    fp = torch.zeros(v.numel() + 1, dtype=torch.int64, device=dev)
                    fp[1:] = torch.cumsum(tk, 0)
                    out = torch.empty(max(int(fp[-1].item()), 1), dtype=torch.int32, device=dev)
                    lrow = (v - self.row0).to(torch.int32).contiguous()
                    kk = r[:, 1].contiguous()
                    dR = torch.tensor([v.numel()], dtype=torch.int64, device=dev)
                    _lib.check(L.gb_sage_sample_keyed(
                        self.tables.handle, v.numel(), _lib.ptr(dR), _lib.ptr(lrow), _lib.ptr(d),
                        _lib.ptr(fp), _lib.ptr(kk), _lib.ptr(self.brp), _lib.ptr(self.bcol), s,
                        seed, epoch, depth, _lib.ptr(out), _lib.stream_ptr()),
                        "gb_sage_sample_keyed")
                    replies[p] = out[: int(fp[-1].item())]
                    if self.ledger is not None and p != self.rank:
                        self.ledger.charge(self.rank, "row-data", 1, replies[p].numel())
            tsel = take_all[sel]
            want = int(tsel.sum().item()) if sel.numel() else 0
            if owner != self.rank:
                self.stats["fetch_ids"] += sel.numel()
                self.stats["fetch_words"] += want + 2 * sel.numel()
                if self.ledger is not None and sel.numel():
                    self.ledger.charge(self.rank, "gather-cols", 1, 2 * sel.numel())
            got = exchange(replies, {owner: want}, self.col_ranks, torch.int32, dev)
            if want:
                # each selected row's picks into its frontier slot
                soff = torch.zeros(sel.numel() + 1, dtype=torch.int64, device=dev)
                soff[1:] = torch.cumsum(tsel, 0)
                _lib.check(L.gb_segment_copy(sel.numel(), _lib.ptr(sel.contiguous()),
                                             _lib.ptr(soff), None, _lib.ptr(got[owner]),
                                             _lib.ptr(fptr), _lib.ptr(fcol), _lib.stream_ptr()),
                           "gb_segment_copy")

    # -- owner sampling over peer memory ----------------------------------------------------
    def _p2p_buffers(self, k):
        """Symmetric-memory frontiers of every layer (same sizes on all ranks):
        rows / batch offsets / frontier offsets / picks, rendezvoused once."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        torch = _torch()
        if self._p2p is not None and self._p2p["k"] == k:
            return self._p2p
        grp = dist.group.WORLD.group_name

        def sym(numel, dtype):
            t = symm_mem.empty(max(int(numel), 1), dtype=dtype, device=self.dev)
            t.zero_()
            return t, symm_mem.rendezvous(t, grp)

        r = k * self.b
        bufs = {"k": k, "layers": []}
        rows, rows_h = sym(r + _lib.GB_COL_PAD, torch.int32)
        brow, brow_h = sym(k + 1, torch.int64)
        for s in self.fanouts:
            fptr, fptr_h = sym(r + 1, torch.int64)
            fcol, fcol_h = sym(r * s + _lib.GB_COL_PAD, torch.int32)
            nbrow, nbrow_h = sym(k + 1, torch.int64)
            bufs["layers"].append({"cap": r, "rows": rows, "rows_h": rows_h, "brow": brow,
                                   "brow_h": brow_h, "fptr": fptr, "fptr_h": fptr_h,
                                   "fcol": fcol, "fcol_h": fcol_h})
            rows, rows_h, brow, brow_h = fcol, fcol_h, nbrow, nbrow_h
            r *= s
        bufs["barrier"] = bufs["layers"][0]["brow_h"]
        L = _lib.lib()
        bufs["ws"] = torch.empty(max(L.gb_sage_owner_p2p_workspace(r), 1), dtype=torch.uint8,
                                 device=self.dev)
        self._p2p = bufs
        return bufs

    def sample_p2p(self, group_batches, epoch, batch_offset, seed):
        """1.5D SAGE with the owner exchange fused into the sampling kernels
        (gb_sage_owner_p2p): per layer, publish rows / offsets, barrier, every
        block owner samples the rows of its block for all grid rows of its
        column straight out of their memory and stores the picks into every
        replica's frontier, barrier, extraction.  No NCCL messages and no
        host synchronisation inside the bulk."""
        import ctypes

        import torch.distributed as dist

        torch = _torch()
        L = _lib.lib()
        grid, st, c = self.grid, self.grid.stages, self.grid.c
        k = len(group_batches)
        bufs = self._p2p_buffers(k)
        off = np.zeros(k + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in group_batches])
        lay0 = bufs["layers"][0]
        if off[-1] > lay0["cap"]:
            raise ContractViolation("more batch vertices than the p2p buffers hold")
        lay0["brow"][: k + 1].copy_(torch.as_tensor(off))
        if off[-1]:
            lay0["rows"][: int(off[-1])].copy_(torch.as_tensor(
                np.concatenate(group_batches).astype(np.int32)))
        # batch offsets of every rank (keys of the rows an owner samples) and
        # the equal-group check the symmetric buffers rely on
        boffs = torch.zeros(grid.p + 1, dtype=torch.int64, device=self.dev)
        boffs[self.rank] = batch_offset
        boffs[grid.p] = k
        kmax = boffs[grid.p:].clone()
        _all_reduce(boffs)
        _all_reduce(kmax, op=dist.ReduceOp.MAX)
        boffs, kmax = boffs.tolist(), int(kmax.item())
        if boffs[grid.p] != k * grid.p or kmax != k:
            raise ContractViolation("fetch='p2p' needs the same number of batches on every grid row")
        owner = self.j * st <= self.i < (self.j + 1) * st
        lo, hi = int(self.bounds[self.i]), int(self.bounds[self.i + 1])
        req = [grid.rank(g, self.j) for g in range(grid.rows)]
        P = ctypes.c_void_p
        barrier = bufs["barrier"]
        layers, stride = [], self.b
        xws = torch.empty(max(L.gb_sage_layer_extract_workspace(self.n, k), 1), dtype=torch.uint8,
                          device=self.dev)
        ws_scan = None
        for l, s in enumerate(self.fanouts):
            if l:
                stride *= self.fanouts[l - 1]
            lay = bufs["layers"][l]
            cap = lay["cap"]
            deg = self.gdeg[lay["rows"][:cap].long()].contiguous()
            if ws_scan is None or ws_scan.numel() * 8 < L.gb_scan_workspace_bytes(cap + 1):
                ws_scan = torch.empty(max(L.gb_scan_workspace_bytes(cap + 1) // 8, 1),
                                      dtype=torch.int64, device=self.dev)
            _lib.check(L.gb_take_scan(cap, _lib.ptr(lay["brow"][k:]), _lib.ptr(deg), s,
                                      _lib.ptr(lay["fptr"]), _lib.ptr(ws_scan),
                                      _lib.stream_ptr()), "gb_take_scan")
            barrier.barrier(channel=0)  # rows, offsets and frontier offsets published
            if owner:
                ng = len(req)
                rows = (P * ng)(*[lay["rows_h"].buffer_ptrs[r] for r in req])
                brow = (P * ng)(*[lay["brow_h"].buffer_ptrs[r] for r in req])
                fptr = (P * ng)(*[lay["fptr_h"].buffer_ptrs[r] for r in req])
                boff = (ctypes.c_int64 * ng)(*[boffs[r] for r in req])
                dst = (P * (ng * c))(*[lay["fcol_h"].buffer_ptrs[grid.rank(g, m)]
                                       for g in range(grid.rows) for m in range(c)])
                ws = bufs["ws"]
                _lib.check(L.gb_sage_owner_p2p(
                    self.tables.handle, ng, rows, brow, fptr, boff, k, cap, c, dst, lo, hi,
                    _lib.ptr(self.brp), _lib.ptr(self.bcol), s, stride, seed, epoch, l + 1,
                    _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "gb_sage_owner_p2p")
            barrier.barrier(channel=0)  # every pick stored
            nxt = bufs["layers"][l + 1]["brow"] if l + 1 < len(self.fanouts) else \
                torch.empty(k + 1, dtype=torch.int64, device=self.dev)
            F_cap = cap * s
            acol = torch.empty(F_cap, dtype=torch.int32, device=self.dev)
            colv = torch.empty(F_cap, dtype=torch.int32, device=self.dev)
            coloff = torch.empty(k + 1, dtype=torch.int64, device=self.dev)
            sizes = torch.zeros(3, dtype=torch.int64, device=self.dev)
            _lib.check(L.gb_sage_layer_extract(self.n, k, _lib.ptr(lay["brow"]),
                                               _lib.ptr(lay["fptr"]), _lib.ptr(lay["fcol"]),
                                               F_cap, _lib.ptr(acol), _lib.ptr(colv),
                                               _lib.ptr(nxt), _lib.ptr(coloff), _lib.ptr(sizes),
                                               _lib.ptr(xws), xws.numel(), _lib.stream_ptr()),
                       "gb_sage_layer_extract")
            layers.append((lay, acol, colv, coloff, nxt, sizes))
        # one host read of the sizes for the reference-shaped views
        sz = torch.stack([x[5] for x in layers]).cpu().numpy()
        out = []
        for (lay, acol, colv, coloff, nxt, _), (R, F, U) in zip(layers, sz):
            R, F, U = int(R), int(F), int(U)
            out.append({
                "frontier_shape": (R, self.n), "frontier_ptr": lay["fptr"][: R + 1],
                "frontier_col": lay["fcol"][:F], "adj_shape": (R, U),
                "adj_ptr": lay["fptr"][: R + 1], "adj_col": acol[:F],
                "rowv_off": lay["brow"][: k + 1], "rowv_cat": lay["rows"][:R],
                "colv_off": coloff, "colv_cat": colv[:U], "sampv_off": nxt, "sampv_cat":
                lay["fcol"][:F]})
        return out

    # -- batch split over the replicas, rows from peer memory ----------------------------
    def batch_slice(self, k):
        """This replica's share [j0, j1) of its grid row's k batches."""
        b = _bounds(k, self.grid.c)
        return int(b[self.j]), int(b[self.j + 1])

    def _peer_table(self):
        """Device block table of the peer row source: bounds and the CSR
        pointers of every block in the owner of this rank's column."""
        torch = _torch()
        if getattr(self, "_ptab", None) is None:
            pb = self._peer_block()
            owners = [self.grid.rank(b, self.j) for b in range(self.grid.rows)]
            self._ptab = (
                torch.as_tensor(np.asarray(self.bounds, np.int64)).to(self.dev),
                torch.tensor([pb["rp_h"].buffer_ptrs[o] for o in owners], dtype=torch.int64,
                             device=self.dev),
                torch.tensor([pb["cl_h"].buffer_ptrs[o] for o in owners], dtype=torch.int64,
                             device=self.dev))
        return self._ptab

    def sample_split(self, group_batches, epoch, batch_offset, seed):
        """1.5D SAGE with the grid row's batches split over its c replicas:
        each runs the single-GPU bulk (dedup Alg. 1: pick in vertex-group
        order, distinct rows staged on chip) with every distinct A row read
        straight from its block owner's memory by the serve kernels.  No
        messages; outputs are this replica's batch slice."""
        from .engine import SageBulk

        torch = _torch()
        j0, j1 = self.batch_slice(len(group_batches))
        mine = [np.asarray(x) for x in group_batches[j0:j1]]
        k = len(mine)
        off = np.zeros(k + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in mine])
        r1 = max(int(off[-1]), 1)
        key = (k, r1)
        if getattr(self, "_split_bulk", None) is None or self._split_key != key:
            self._split_bulk = SageBulk(self.tables, max(k, 1), max(k * self.b, r1), self.b,
                                        self.fanouts, mode="dedup")
            self._split_key = key
        d_off = torch.as_tensor(off).to(self.dev)
        d_cat = torch.as_tensor(np.concatenate(mine).astype(np.int32) if off[-1]
                                else np.zeros(1, np.int32)).to(self.dev)
        if not k:
            return []
        bulk = self._split_bulk
        bulk.launch_peer(d_off, d_cat, seed, epoch, batch_offset + j0, self._peer_table())
        return [ls.device for ls in bulk.layers(d_off, d_cat)]

    # -- one bulk --------------------------------------------------------------------------
    def sample(self, group_batches, epoch, batch_offset, seed):
        """Sample this grid row's group; returns (device layer dicts, sizes)."""
        if self.fetch == "p2p":
            return self.sample_p2p(group_batches, epoch, batch_offset, seed)
        if self.fetch == "split":
            return self.sample_split(group_batches, epoch, batch_offset, seed)
        import torch.distributed as dist

        torch = _torch()
        L = _lib.lib()
        k = len(group_batches)
        off = np.zeros(k + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in group_batches])
        brow = torch.as_tensor(off).to(self.dev)
        rowv = torch.as_tensor(np.concatenate(group_batches).astype(np.int32) if k and off[-1]
                               else np.zeros(1, np.int32)).to(self.dev)
        R = int(off[-1])
        stride = self.b
        layers = []
        ws_scan = torch.empty(max(L.gb_scan_workspace_bytes(1 + R * int(np.prod(self.fanouts)))
                                  // 8, 1), dtype=torch.int64, device=self.dev)
        for l, s in enumerate(self.fanouts):
            if l:
                stride *= self.fanouts[l - 1]
            rv = rowv[:R]
            deg = self.gdeg[rv.long()] if R else torch.zeros(0, dtype=torch.int32,
                                                             device=self.dev)
            fptr = torch.empty(R + 1, dtype=torch.int64, device=self.dev)
            dR = torch.tensor([R], dtype=torch.int64, device=self.dev)
            _lib.check(L.gb_take_scan(max(R, 1), _lib.ptr(dR), _lib.ptr(deg if R else None), s,
                                      _lib.ptr(fptr), _lib.ptr(ws_scan), _lib.stream_ptr()),
                       "gb_take_scan")
            F = int(fptr[R].item())
            mine = (rv >= self.V0) & (rv < self.V1)
            fcol = torch.zeros(max(F, 1), dtype=torch.int32, device=self.dev)
            if self.fetch == "owner":
                self.owner_sample(rv, mine, deg, fptr, brow, k, stride, batch_offset, s, seed,
                                  epoch, l + 1, fcol)
            else:
                U = torch.unique(rv[mine])
                t0 = self._phase(None, 0.0)
                lrowptr, lcol = self.fetch_rows(U)
                self._phase("fetch", t0)
                lrow = torch.searchsorted(U, rv).to(torch.int32)
                deg_mine = torch.where(mine, deg, torch.zeros_like(deg)).contiguous()
                ws = torch.empty(max(L.gb_sage_layer_sample_workspace(max(R, 1), max(R, 1) * s),
                                     1), dtype=torch.uint8, device=self.dev)
                mode = _lib.GB_SAGE_STREAM if self.mode == "stream" else _lib.GB_SAGE_PFREE
                if R:
                    _lib.check(L.gb_sage_layer_sample(
                        self.tables.handle, k, _lib.ptr(brow), R, _lib.ptr(lrow),
                        _lib.ptr(deg_mine), _lib.ptr(fptr), _lib.ptr(lrowptr), _lib.ptr(lcol), s,
                        stride, batch_offset, seed, epoch, l + 1, mode, _lib.ptr(fcol),
                        _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "gb_sage_layer_sample")
            # step 2: sample-then-reduce inside the grid row
            if self.grid.c > 1 and F:
                t0 = self._phase(None, 0.0)
                _all_reduce(fcol[:F], op=dist.ReduceOp.SUM,
                                group=self.row_groups[self.i])
                self._phase("reduce", t0)
                self.stats["reduce_words"] += F
                if self.ledger is not None:
                    self.ledger.charge(self.rank, "all-reduce", 1, F)
            # step 3: extraction on the complete frontier
            acol = torch.empty(max(F, 1), dtype=torch.int32, device=self.dev)
            colv = torch.empty(max(F, 1), dtype=torch.int32, device=self.dev)
            eoff = torch.empty(k + 1, dtype=torch.int64, device=self.dev)
            coloff = torch.empty(k + 1, dtype=torch.int64, device=self.dev)
            sizes = torch.zeros(3, dtype=torch.int64, device=self.dev)
            xws = torch.empty(max(L.gb_sage_layer_extract_workspace(self.n, k), 1),
                              dtype=torch.uint8, device=self.dev)
            _lib.check(L.gb_sage_layer_extract(self.n, k, _lib.ptr(brow), _lib.ptr(fptr),
                                               _lib.ptr(fcol), max(F, 1), _lib.ptr(acol),
                                               _lib.ptr(colv), _lib.ptr(eoff), _lib.ptr(coloff),
                                               _lib.ptr(sizes), _lib.ptr(xws), xws.numel(),
                                               _lib.stream_ptr()), "gb_sage_layer_extract")
            U_tot = int(sizes[2].item())
            layers.append({
                "frontier_shape": (R, self.n), "frontier_ptr": fptr, "frontier_col": fcol[:F],
                "adj_shape": (R, U_tot), "adj_ptr": fptr, "adj_col": acol[:F],
                "rowv_off": brow, "rowv_cat": rowv[:R], "colv_off": coloff,
                "colv_cat": colv[:U_tot], "sampv_off": eoff, "sampv_cat": fcol[:F],
            })
            rowv, brow, R = fcol, eoff, F
        return layers


class Ladies15D(Sage15D):
    def sample_p2p(self, group_batches, epoch, batch_offset, seed):
        """1.5D LADIES with the replicas of a grid row splitting its batches:
        each layer gathers the A rows of its Q straight from the block
        owners' memory (peer reads) and runs the single-GPU race layer on them
        (gb_ladies_layer_rows: column tiles in shared memory, keys, radix
        select, extraction).  The partial-count merge and candidate exchange
        of the message-based variant disappear: every sampled set is complete
        where it is computed."""
        torch = _torch()
        L = _lib.lib()
        dev, n = self.dev, self.n
        j0, j1 = self.batch_slice(len(group_batches))
        mine = group_batches[j0:j1]
        k = len(mine)
        off = np.zeros(k + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in mine])
        qoff = torch.as_tensor(off).to(dev)
        qcol = torch.as_tensor(np.concatenate([np.sort(np.asarray(x)) for x in mine])
                               .astype(np.int32) if off[-1] else np.zeros(1, np.int32)).to(dev)
        layers = []
        prof = os.environ.get("GB_PROF15") == "1"
        tp = {}

        def mark(name, t0=[None]):
            if not prof:
                return
            torch.cuda.synchronize()
            t = time.perf_counter()
            if t0[0] is not None:
                tp[name] = tp.get(name, 0.0) + (t - t0[0]) * 1e3
            t0[0] = t

        mark("start")
        for l, s in enumerate(self.fanouts):
            QN = int(qoff[k].item()) if k else 0
            qc = qcol[:QN]
            U = torch.unique(qc)
            mark("unique")
            lrowptr, lcol = self.fetch_rows_any(U)
            mark("fetch")
            lrow = torch.searchsorted(U, qc).to(torch.int32).contiguous()
            qcap = max(QN, 1)
            o = {"fptr": torch.zeros(k + 1, dtype=torch.int64, device=dev),
                 "fcol": torch.zeros(max(k * s, 1), dtype=torch.int32, device=dev),
                 "aptr": torch.zeros(qcap + 1, dtype=torch.int64, device=dev),
                 "acol": torch.zeros(qcap * s, dtype=torch.int32, device=dev),
                 "coloff": torch.zeros(k + 1, dtype=torch.int64, device=dev)}
            out = _lib.LadiesLayerOut()
            for name in ("fptr", "fcol", "aptr", "acol", "coloff"):
                setattr(out, name, o[name].data_ptr())
            out.q_cap, out.f_cap, out.a_cap = qcap, max(k * s, 1), qcap * s
            sizes = torch.zeros(5, dtype=torch.int64, device=dev)
            fan = (ctypes.c_int64 * 1)(s)
            wsb = ctypes.c_size_t()
            _lib.check(L.gb_ladies_bulk_workspace(self.tables.handle, max(k, 1), qcap, 1, fan,
                                                  _lib.GB_LADIES_RACE, ctypes.byref(wsb)),
                       "gb_ladies_bulk_workspace")
            ws = torch.empty(max(int(wsb.value), 1), dtype=torch.uint8, device=dev)
            mark("alloc")
            if k:
                _lib.check(L.gb_ladies_layer_rows(
                    self.tables.handle, k, _lib.ptr(qoff), _lib.ptr(lrow), qcap, _lib.ptr(lrowptr),
                    _lib.ptr(lcol), s, seed, epoch, l + 1, batch_offset + j0,
                    _lib.GB_LADIES_RACE, ctypes.byref(out), _lib.ptr(sizes), _lib.ptr(ws),
                    ws.numel(), _lib.stream_ptr()), "gb_ladies_layer_rows")
            mark("layer")
            R, F, A, C = (int(x) for x in sizes.tolist()[:4])
            layers.append({
                "frontier_shape": (k, n), "frontier_ptr": o["fptr"], "frontier_col": o["fcol"][:F],
                "adj_shape": (QN, C), "adj_ptr": o["aptr"][: QN + 1], "adj_col": o["acol"][:A],
                "rowv_off": qoff, "rowv_cat": qc,
                "colv_off": o["fptr"], "colv_cat": o["fcol"][:F],
                "sampv_off": o["fptr"], "sampv_cat": o["fcol"][:F]})
            qoff, qcol = o["fptr"], o["fcol"]
            mark("sizes")
        if prof and self.rank == 0:
            print("GB_PROF15 ladies p2p ms:", {a: round(b, 3) for a, b in tp.items()},
                  file=sys.stderr)
        return layers

    """1.5D partitioned LADIES (exponential-race sampling) over real processes.

    Per layer, grid row i (k_i batches), replica j:
      1. row fetch of the batch vertices in column j's range (as SAGE);
      2. partial P: counts e_v from the fetched rows (gb_ladies_counts);
      3. sparse merge (reduce-scatter by vertex range over the c replicas):
         replica m receives every (batch, v, e) with v in its range and sums
         them, so it owns the exact counts of its vertices;
      4. local top-s by race key (gb_ladies_race_topk), all-gather of the
         c*s candidates, final top-s by (key, v) — keys depend only on
         (batch, v, e), so the result equals the single-GPU race sampler;
      5. A_S rows for the replica's own Q vertices in the slot layout
         (gb_ladies_extract_rows), summed over the grid row (C4, dist.py:523).
    """

    def sample(self, group_batches, epoch, batch_offset, seed):
        import torch.distributed as dist

        if self.fetch == "p2p":
            return self.sample_p2p(group_batches, epoch, batch_offset, seed)
        torch = _torch()
        L = _lib.lib()
        dev, n, c = self.dev, self.n, self.grid.c
        k = len(group_batches)
        rg = self.row_groups[self.i]
        off = np.zeros(k + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in group_batches])
        qoff = torch.as_tensor(off).to(dev)
        qcol = torch.as_tensor(np.concatenate([np.sort(np.asarray(x)) for x in group_batches])
                               .astype(np.int32) if off[-1] else np.zeros(0, np.int32)).to(dev)
        vr = _bounds(n, c)
        layers = []
        for l, s in enumerate(self.fanouts):
            QN = int(qoff[k].item())
            qc = qcol[:QN]
            mine = (qc >= self.V0) & (qc < self.V1)
            U = torch.unique(qc[mine])
            lrowptr, lcol = self.fetch_rows(U)
            nnz = int(lrowptr[-1].item())
            lrowptr = torch.cat([lrowptr, lrowptr[-1:]])  # dummy empty row U.numel()
            lrow = torch.searchsorted(U, qc).to(torch.int32)
            lrow = torch.where(mine, lrow, torch.full_like(lrow, U.numel())).contiguous()
            qdeg = torch.where(mine, self.gdeg[qc.long()], torch.zeros_like(lrow)).contiguous()
            # -- partial counts
            pcap = max(min(k * n, int(qdeg.long().sum().item())), 1)
            poff = torch.zeros(k + 1, dtype=torch.int64, device=dev)
            pv = torch.empty(pcap, dtype=torch.int32, device=dev)
            pe = torch.empty(pcap, dtype=torch.int32, device=dev)
            ws = torch.empty(max(L.gb_ladies_counts_workspace(k, n, max(QN, 1)), 1),
                             dtype=torch.uint8, device=dev)
            _lib.check(L.gb_ladies_counts(k, _lib.ptr(qoff), _lib.ptr(lrow), _lib.ptr(qdeg),
                                          max(QN, 1), _lib.ptr(lrowptr), _lib.ptr(lcol), n,
                                          _lib.ptr(poff), _lib.ptr(pv), _lib.ptr(pe),
                                          _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
                       "gb_ladies_counts")
            P = int(poff[k].item())
            bid = torch.repeat_interleave(torch.arange(k, device=dev, dtype=torch.int32),
                                          (poff[1:] - poff[:-1]))
            trip = torch.stack([bid, pv[:P], pe[:P]], 1)
            # -- sparse merge: reduce-scatter by vertex range inside the grid row
            sends = {}
            for m in range(c):
                sel = (trip[:, 1] >= int(vr[m])) & (trip[:, 1] < int(vr[m + 1]))
                sends[self.grid.rank(self.i, m)] = trip[sel].flatten().contiguous()
            cnts = exchange_counts(sends, self.row_ranks, dev)
            got = exchange(sends, cnts, self.row_ranks, torch.int32, dev)
            allt = torch.cat([got[p].view(-1, 3) for p in self.row_ranks if p in got]) \
                if got else torch.zeros((0, 3), dtype=torch.int32, device=dev)
            # sum the partials of this replica's vertex range on the device
            v0, v1 = int(vr[self.j]), int(vr[self.j + 1])
            allt = allt.contiguous()
            mcnt = allt.shape[0]
            moff = torch.zeros(k + 1, dtype=torch.int64, device=dev)
            mv = torch.empty(max(mcnt, 1), dtype=torch.int32, device=dev)
            me = torch.empty(max(mcnt, 1), dtype=torch.int32, device=dev)
            mws = torch.empty(max(L.gb_ladies_merge_counts_workspace(k, v1 - v0), 1),
                              dtype=torch.uint8, device=dev)
            _lib.check(L.gb_ladies_merge_counts(k, mcnt, _lib.ptr(allt), v0, v1 - v0,
                                                _lib.ptr(moff), _lib.ptr(mv), _lib.ptr(me),
                                                _lib.ptr(mws), mws.numel(), _lib.stream_ptr()),
                       "gb_ladies_merge_counts")
            # -- local race top-s, then the grid-row merge of candidates
            mcap = max(mv.numel(), 1)
            take = torch.zeros(k, dtype=torch.int64, device=dev)
            Sv = torch.zeros(max(k * s, 1), dtype=torch.int32, device=dev)
            Sk = torch.zeros(max(k * s, 1), dtype=torch.int32, device=dev)
            rws = torch.empty(max(L.gb_ladies_race_topk_workspace(k, mcap, s), 1),
                              dtype=torch.uint8, device=dev)
            if k:
                _lib.check(L.gb_ladies_race_topk(k, _lib.ptr(moff), _lib.ptr(mv), _lib.ptr(me),
                                                 mcap, s, seed, epoch, l + 1, batch_offset,
                                                 _lib.ptr(take), _lib.ptr(Sv), _lib.ptr(Sk),
                                                 _lib.ptr(rws), rws.numel(), _lib.stream_ptr()),
                           "gb_ladies_race_topk")
            nb = (moff[1:] - moff[:-1]).clone()
            if c > 1:
                _all_reduce(nb, group=rg)
                pack = torch.cat([take, Sv[:k * s].long(), (Sk[:k * s].long() & 0xffffffff)])
                parts = [torch.empty_like(pack) for _ in range(c)]
                _all_gather(parts, pack, group=rg)
            else:
                parts = [torch.cat([take, Sv[:k * s].long(), Sk[:k * s].long() & 0xffffffff])]
            ct, cv, ck, cb = [], [], [], []
            for pt in parts:
                tk = pt[:k]
                v2 = pt[k:k + k * s].view(k, s)
                k2 = pt[k + k * s:].view(k, s)
                valid = torch.arange(s, device=dev)[None, :] < tk[:, None]
                cv.append(v2[valid])
                ck.append(k2[valid])
                cb.append(torch.arange(k, device=dev)[:, None].expand(k, s)[valid])
            cv, ck, cb = torch.cat(cv), torch.cat(ck), torch.cat(cb)
            o1 = torch.argsort(cv, stable=True)
            o2 = torch.argsort((cb[o1] << 32) | ck[o1], stable=True)
            order = o1[o2]
            cb, cv = cb[order], cv[order]
            tk = torch.minimum(nb, torch.full_like(nb, s))
            first = torch.zeros(k + 1, dtype=torch.int64, device=dev)
            first[1:] = torch.cumsum(torch.bincount(cb, minlength=k), 0)
            rank = torch.arange(cb.numel(), device=dev) - first[cb]
            keep = rank < tk[cb]
            fb, fv = cb[keep], cv[keep]
            o3 = torch.argsort((fb << 32) | fv)
            fcol = fv[o3].to(torch.int32).contiguous()
            fptr = torch.zeros(k + 1, dtype=torch.int64, device=dev)
            fptr[1:] = torch.cumsum(tk, 0)
            F = int(fptr[k].item())
            # -- extraction of this replica's Q rows, summed over the grid row
            takes = tk
            shared = bool((takes == takes[0]).all().item()) if k else True
            coloff = torch.zeros(k + 1, dtype=torch.int64, device=dev) if shared else fptr.clone()
            qb = torch.repeat_interleave(torch.arange(k, device=dev), qoff[1:] - qoff[:-1])
            rcap = torch.minimum(self.gdeg[qc.long()].long(), takes[qb]) if QN else \
                torch.zeros(0, dtype=torch.int64, device=dev)
            slot = torch.zeros(QN + 1, dtype=torch.int64, device=dev)
            slot[1:] = torch.cumsum(rcap, 0)
            slots = torch.zeros(max(int(slot[-1].item()), 1), dtype=torch.int32, device=dev)
            rcnt = torch.zeros(max(QN, 1), dtype=torch.int32, device=dev)
            if QN:
                _lib.check(L.gb_ladies_extract_rows(k, _lib.ptr(qoff), _lib.ptr(lrow),
                                                    _lib.ptr(lrowptr), _lib.ptr(lcol),
                                                    _lib.ptr(fptr), _lib.ptr(fcol),
                                                    _lib.ptr(coloff), _lib.ptr(slot),
                                                    _lib.ptr(slots), _lib.ptr(rcnt),
                                                    _lib.stream_ptr()), "gb_ladies_extract_rows")
            if c > 1 and QN:
                _all_reduce(slots, group=rg)
                _all_reduce(rcnt, group=rg)
                self.stats["reduce_words"] += slots.numel() + rcnt.numel()
            aptr = torch.zeros(QN + 1, dtype=torch.int64, device=dev)
            aptr[1:] = torch.cumsum(rcnt[:QN].long(), 0)
            E = int(aptr[-1].item())
            acol = torch.zeros(max(E, 1), dtype=torch.int32, device=dev)
            if E:
                _lib.check(L.gb_segment_copy(QN, None, _lib.ptr(slot), _lib.ptr(rcnt),
                                             _lib.ptr(slots), _lib.ptr(aptr), _lib.ptr(acol),
                                             _lib.stream_ptr()), "gb_segment_copy")
            acol = acol[:E]
            width = 0 if k == 0 else (int(takes[0].item()) if shared else F)
            layers.append({
                "frontier_shape": (k, n), "frontier_ptr": fptr, "frontier_col": fcol,
                "adj_shape": (QN, width), "adj_ptr": aptr, "adj_col": acol,
                "rowv_off": qoff, "rowv_cat": qc, "colv_off": fptr, "colv_cat": fcol,
                "sampv_off": fptr, "sampv_cat": fcol,
            })
            del nnz
            qoff, qcol = fptr, fcol
        return layers


def ladies_epoch_15d(sampler: Ladies15D, cfg, batches, epoch=0, batch_offset=0):
    """Distributed LADIES epoch over the grid, gathered on every rank."""
    import torch.distributed as dist

    from .dist import merge_epochs

    grid = sampler.grid
    b = _bounds(len(batches), grid.rows)
    g0, g1 = int(b[sampler.i]), int(b[sampler.i + 1])
    mine = sampler.sample([np.asarray(x) for x in batches[g0:g1]], epoch, batch_offset + g0,
                          cfg.seed)
    local = [{k2: (v if isinstance(v, tuple) else v.cpu().numpy()) for k2, v in lay.items()}
             for lay in mine]
    allp = [None] * grid.p
    dist.all_gather_object(allp, local)
    parts = []
    for i in range(grid.rows):
        gi = [np.asarray(x) for x in batches[int(b[i]):int(b[i + 1])]]
        if sampler.fetch == "p2p":  # the grid row's batches split over its replicas
            cb = _bounds(len(gi), grid.c)
            for j in range(grid.c):
                if int(cb[j + 1]) == int(cb[j]):
                    continue
                parts.append(SampledEpoch(SamplerKind.LADIES, epoch, gi[int(cb[j]):int(cb[j + 1])],
                                          [LayerSample(d + 1, device=x, n=sampler.n)
                                           for d, x in enumerate(allp[grid.rank(i, j)])],
                                          cfg.layers))
            continue
        parts.append(SampledEpoch(SamplerKind.LADIES, epoch, gi,
                                  [LayerSample(d + 1, device=x, n=sampler.n)
                                   for d, x in enumerate(allp[grid.rank(i, 0)])], cfg.layers))
    return merge_epochs(SamplerKind.LADIES, epoch, batches, parts, cfg.layers)


def sage_epoch_15d(sampler: Sage15D, cfg, batches, epoch=0, batch_offset=0, gather=True):
    """Distributed SAGE epoch: grid row i samples group i; with gather=True
    every rank returns the full epoch (groups gathered over the grid column
    and concatenated — identical to the serial epoch)."""
    import torch.distributed as dist

    from .dist import merge_epochs

    grid = sampler.grid
    b = _bounds(len(batches), grid.rows)
    g0, g1 = int(b[sampler.i]), int(b[sampler.i + 1])
    mine = sampler.sample([np.asarray(x) for x in batches[g0:g1]], epoch, batch_offset + g0,
                          cfg.seed)
    if not gather:
        return mine
    local = [{k: (v if isinstance(v, tuple) else v.cpu().numpy()) for k, v in lay.items()}
             for lay in mine]
    allp = [None] * grid.p
    dist.all_gather_object(allp, local)
    parts = []
    for i in range(grid.rows):
        gi = [np.asarray(x) for x in batches[int(b[i]):int(b[i + 1])]]
        if sampler.fetch == "split":  # the grid row's batches split over its replicas
            cb = _bounds(len(gi), grid.c)
            for j in range(grid.c):
                if int(cb[j + 1]) == int(cb[j]):
                    continue
                parts.append(SampledEpoch(SamplerKind.SAGE, epoch, gi[int(cb[j]):int(cb[j + 1])],
                                          [LayerSample(d + 1, device=x, n=sampler.n)
                                           for d, x in enumerate(allp[grid.rank(i, j)])],
                                          cfg.layers))
            continue
        lay = allp[grid.rank(i, 0)]
        parts.append(SampledEpoch(SamplerKind.SAGE, epoch, gi,
                                  [LayerSample(d + 1, device=x, n=sampler.n)
                                   for d, x in enumerate(lay)], cfg.layers))
    return merge_epochs(SamplerKind.SAGE, epoch, batches, parts, cfg.layers)


def fetch_features_nccl(vertices, H_block, row_starts, grid: ProcessGrid, group_col_ranks):
    """fetch_features (pipeline.py:78-120) over real processes: every rank
    requests the fp32 feature rows of `vertices` from the replicas in its own
    grid column (block row owner (r, j)), served by gb_gather_features and
    delivered by a grouped send/recv all-to-allv.  Returns rows in request
    order (duplicates fetched per occurrence)."""
    import torch.distributed as dist

    torch = _torch()
    me = dist.get_rank()
    i, j = grid.coords(me)
    dev = H_block.device
    f = H_block.shape[1]
    v = torch.as_tensor(np.asarray(vertices, np.int64)).to(dev)
    rs = torch.as_tensor(np.asarray(row_starts, np.int64)).to(dev)
    owner_row = torch.searchsorted(rs, v, right=True) - 1
    sends, slots = {}, {}
    for r in range(grid.rows):
        sel = torch.nonzero(owner_row == r).flatten()
        sends[grid.rank(r, j)] = v[sel].to(torch.int32)
        slots[grid.rank(r, j)] = sel
    counts = exchange_counts(sends, group_col_ranks, dev)
    reqs = exchange(sends, counts, group_col_ranks, torch.int32, dev)
    L = _lib.lib()
    replies = {}
    for p, ids in reqs.items():
        buf = torch.empty((ids.numel(), f), dtype=torch.float32, device=dev)
        _lib.check(L.gb_gather_features(ids.numel(), _lib.ptr(ids), int(row_starts[i]),
                                        _lib.ptr(H_block), f, _lib.ptr(buf), _lib.stream_ptr()),
                   "gb_gather_features")
        replies[p] = buf.flatten()
    want = {p: sends[p].numel() * f for p in group_col_ranks}
    got = exchange(replies, want, group_col_ranks, torch.float32, dev)
    out = torch.empty((v.numel(), f), dtype=torch.float32, device=dev)
    for p, sel in slots.items():
        if sel.numel():
            out[sel] = got[p].view(-1, f)
    return out


class PeerFeatures:
    """Feature block rows in symmetric memory: block i (rows row_starts[i] ..
    row_starts[i+1]) on every rank of grid row i, padded to the largest block
    so every rank allocates the same size (torch symmetric memory,
    rendezvoused once over the world group)."""

    def __init__(self, H_block, row_starts, grid: ProcessGrid):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        torch = _torch()
        self.grid = grid
        self.row_starts = np.asarray(row_starts, np.int64)
        self.f = int(H_block.shape[1])
        rows = int(np.max(np.diff(self.row_starts)))
        self.buf = symm_mem.empty(max(rows, 1) * self.f, dtype=torch.float32,
                                  device=H_block.device)
        self.buf[: H_block.numel()].copy_(H_block.flatten())
        self.handle = symm_mem.rendezvous(self.buf, dist.group.WORLD.group_name)
        self.handle.barrier(channel=0)


def fetch_features_p2p(vertices, peer: PeerFeatures):
    """fetch_features (pipeline.py:78-120) with the all-to-allv fused into
    the gather: the requester reads each feature row straight out of the
    block owner's memory in its own grid column (P2P loads over NVLink,
    gb_gather_features on the peer pointer) — no request / reply messages.
    Returns rows in request order (duplicates per occurrence)."""
    import torch.distributed as dist

    torch = _torch()
    grid, f = peer.grid, peer.f
    me = dist.get_rank()
    _, j = grid.coords(me)
    dev = peer.buf.device
    v = torch.as_tensor(np.asarray(vertices, np.int64)).to(dev)
    rs = torch.as_tensor(peer.row_starts).to(dev)
    owner_row = torch.searchsorted(rs, v, right=True) - 1
    out = torch.empty((v.numel(), f), dtype=torch.float32, device=dev)
    L = _lib.lib()
    for r in range(grid.rows):
        sel = torch.nonzero(owner_row == r).flatten()
        if sel.numel() == 0:
            continue
        ids = v[sel].to(torch.int32).contiguous()
        rows = torch.empty((ids.numel(), f), dtype=torch.float32, device=dev)
        src = peer.handle.buffer_ptrs[grid.rank(r, j)]
        _lib.check(L.gb_gather_features(ids.numel(), _lib.ptr(ids), int(peer.row_starts[r]),
                                        ctypes.c_void_p(src), f, _lib.ptr(rows),
                                        _lib.stream_ptr()), "gb_gather_features")
        out[sel] = rows
    return out
