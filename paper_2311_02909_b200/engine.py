"""Device orchestration of the bulk samplers: buffer planning, C-ABI launches,
and conversion of device results into `SampledEpoch` objects.

`SageBulk` owns every buffer of one bulk shape (graph, k, rows, fanouts);
`launch()` is a single host call that enqueues all layers on the current
stream without any host synchronisation, so repeated bulks can be captured
in a CUDA graph (bench.py does).  Results are read back only when
`epoch()` is called.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ContractViolation
from .sampler import LayerSample, SampledEpoch, SamplerConfig, SamplerKind, _flatten_batches
from .sparse import Graph

MODES = {"stream": _lib.GB_SAGE_STREAM, "pfree": _lib.GB_SAGE_PFREE,
         "dedup": _lib.GB_SAGE_DEDUP}


def sage_caps(r1_cap, fanouts):
    """Upper bounds (rows, entries) per layer: R_{l+1} = F_l <= R_l * s_l."""
    caps, r = [], int(r1_cap)
    for s in fanouts:
        caps.append((r, r * int(s)))
        r = r * int(s)
    return caps


class SageBulk:
    """Reusable device buffers + launcher for SAGE bulks of one shape."""

    def __init__(self, dg, k, r1_cap, batch_size, fanouts, mode="dedup"):
        import torch

        self.dg, self.k, self.r1_cap = dg, int(k), int(r1_cap)
        self.batch_size = int(batch_size)
        self.fanouts = tuple(int(s) for s in fanouts)
        if mode not in MODES:
            raise ContractViolation(f"unknown SAGE mode {mode!r}")
        self.mode = mode
        L = len(self.fanouts)
        dev = torch.device("cuda")
        self.caps = sage_caps(self.r1_cap, self.fanouts)
        self.out = []
        self.c_layers = (_lib.SageLayerOut * L)()
        for l, (rc, fc) in enumerate(self.caps):
            o = {
                "fptr": torch.empty(rc + 1, dtype=torch.int64, device=dev),
                "fcol": torch.empty(max(fc, 1), dtype=torch.int32, device=dev),
                "acol": torch.empty(max(fc, 1), dtype=torch.int32, device=dev),
                "colv": torch.empty(max(fc, 1), dtype=torch.int32, device=dev),
                "eoff": torch.empty(self.k + 1, dtype=torch.int64, device=dev),
                "coloff": torch.empty(self.k + 1, dtype=torch.int64, device=dev),
            }
            self.out.append(o)
            c = self.c_layers[l]
            for name in ("fptr", "fcol", "acol", "colv", "eoff", "coloff"):
                setattr(c, name, o[name].data_ptr())
            c.r_cap, c.f_cap = rc, fc
        self.h_fanouts = np.ascontiguousarray(self.fanouts, dtype=np.int64)
        nbytes = ctypes.c_size_t()
        _lib.check(_lib.lib().gb_sage_bulk_workspace(
            dg.handle, self.k, self.r1_cap, L, self.h_fanouts.ctypes.data,
            ctypes.byref(nbytes)), "gb_sage_bulk_workspace")
        # zero-filled once: the library keeps its bit maps and vertex counters
        # clear between bulks on this workspace (gnnbulk_b200.h, gb_sage_bulk)
        self.ws = torch.zeros(max(int(nbytes.value), 1), dtype=torch.uint8, device=dev)
        self.sizes = torch.zeros(3 * L, dtype=torch.int64, device=dev)

    def launch_peer(self, d_bptr, d_bverts, seed, epoch, batch_offset, peer, stream=None):
        """The bulk (dedup mode) with the A rows read from their owners'
        memory: peer = (bounds int64[nblk + 1], brp pointers, bcol pointers)
        as device tensors (gb_sage_bulk_peer)."""
        bounds, brp, bcol = peer
        L = len(self.fanouts)
        _lib.check(_lib.lib().gb_sage_bulk_peer(
            self.dg.handle, self.k, _lib.ptr(d_bptr), _lib.ptr(d_bverts), self.r1_cap,
            self.batch_size, L, self.h_fanouts.ctypes.data, int(seed), int(epoch),
            int(batch_offset), self.c_layers, _lib.ptr(self.sizes), _lib.ptr(self.ws),
            self.ws.numel(), int(bounds.numel() - 1), _lib.ptr(bounds), _lib.ptr(brp),
            _lib.ptr(bcol), _lib.stream_ptr(stream)), "gb_sage_bulk_peer")

    def launch(self, d_bptr, d_bverts, seed, epoch, batch_offset, stream=None):
        """Enqueue the whole bulk (all layers) on `stream`; no host sync."""
        L = len(self.fanouts)
        _lib.check(_lib.lib().gb_sage_bulk(
            self.dg.handle, self.k, _lib.ptr(d_bptr), _lib.ptr(d_bverts), self.r1_cap,
            self.batch_size, L, self.h_fanouts.ctypes.data, int(seed), int(epoch),
            int(batch_offset), MODES[self.mode], self.c_layers, _lib.ptr(self.sizes),
            _lib.ptr(self.ws), self.ws.numel(), _lib.stream_ptr(stream)), "gb_sage_bulk")

    def layers(self, d_bptr, d_bverts, sizes=None):
        """Device-resident LayerSamples (views sized by the per-layer counts)."""
        if sizes is None:
            sizes = self.sizes.cpu().numpy()
        n = self.dg.n
        out = []
        rowv, brow = d_bverts, d_bptr
        for l in range(len(self.fanouts)):
            R, F, U = (int(x) for x in sizes[3 * l: 3 * l + 3])
            o = self.out[l]
            dev = {
                "frontier_shape": (R, n), "frontier_ptr": o["fptr"][: R + 1],
                "frontier_col": o["fcol"][:F],
                "adj_shape": (R, U), "adj_ptr": o["fptr"][: R + 1], "adj_col": o["acol"][:F],
                "rowv_off": brow, "rowv_cat": rowv[:R],
                "colv_off": o["coloff"], "colv_cat": o["colv"][:U],
                "sampv_off": o["eoff"], "sampv_cat": o["fcol"][:F],
            }
            out.append(LayerSample(l + 1, device=dev, n=n))
            rowv, brow = o["fcol"], o["eoff"]
        return out


def upload_batches(batches, n, batch_size=None, sort_within=False):
    """Validate batches on the host (reference _flatten_batches checks) and
    upload (offsets int64, vertices int32)."""
    import torch

    cat, off = _flatten_batches(batches, n, sort_within=sort_within)
    if batch_size is not None and len(batches) and int(np.max(np.diff(off))) > batch_size:
        raise ContractViolation("actual rows exceed the nominal stride")
    d_off = torch.as_tensor(off).cuda()
    d_cat = torch.as_tensor(cat.astype(np.int32)).cuda() if cat.size else torch.zeros(
        1, dtype=torch.int32, device="cuda")
    return d_off, d_cat, int(off[-1])


def sage_epoch(G: Graph, cfg: SamplerConfig, batches, epoch, batch_offset, mode="dedup"):
    dg = G.device()
    d_off, d_cat, r1 = upload_batches(batches, G.n, cfg.batch_size)
    bulk = SageBulk(dg, len(batches), max(r1, 1), cfg.batch_size, cfg.fanouts, mode=mode)
    bulk.launch(d_off, d_cat, cfg.seed, epoch, batch_offset)
    layers = bulk.layers(d_off, d_cat)
    return SampledEpoch(SamplerKind.SAGE, epoch, batches, layers, cfg.layers)


LADIES_MODES = {"exact": _lib.GB_LADIES_EXACT, "race": _lib.GB_LADIES_RACE,
                "race_dense": _lib.GB_LADIES_RACE_DENSE}
# auto -> exact replay while its O(s * N) serial cumsum per batch stays small
LADIES_EXACT_LIMIT = 1 << 26


class LadiesBulk:
    """Reusable device buffers + launcher for LADIES bulks of one shape."""

    def __init__(self, dg, k, q1_cap, fanouts, mode="race"):
        import torch

        if mode not in LADIES_MODES:
            raise ContractViolation(f"unknown LADIES mode {mode!r}")
        self.dg, self.k, self.q1_cap = dg, int(k), int(q1_cap)
        self.fanouts = tuple(int(s) for s in fanouts)
        self.mode = mode
        L = len(self.fanouts)
        dev = torch.device("cuda")
        self.out = []
        self.c_layers = (_lib.LadiesLayerOut * L)()
        qc = self.q1_cap
        for l, s in enumerate(self.fanouts):
            fc, ac = self.k * s, qc * s
            o = {
                "fptr": torch.empty(self.k + 1, dtype=torch.int64, device=dev),
                "fcol": torch.empty(max(fc, 1), dtype=torch.int32, device=dev),
                "aptr": torch.empty(qc + 1, dtype=torch.int64, device=dev),
                "acol": torch.empty(max(ac, 1), dtype=torch.int32, device=dev),
                "coloff": torch.empty(self.k + 1, dtype=torch.int64, device=dev),
            }
            self.out.append(o)
            c = self.c_layers[l]
            for name in ("fptr", "fcol", "aptr", "acol", "coloff"):
                setattr(c, name, o[name].data_ptr())
            c.q_cap, c.f_cap, c.a_cap = qc, fc, ac
            qc = fc
        self.h_fanouts = np.ascontiguousarray(self.fanouts, dtype=np.int64)
        nbytes = ctypes.c_size_t()
        _lib.check(_lib.lib().gb_ladies_bulk_workspace(
            dg.handle, self.k, self.q1_cap, L, self.h_fanouts.ctypes.data, LADIES_MODES[mode],
            ctypes.byref(nbytes)), "gb_ladies_bulk_workspace")
        self.ws = torch.empty(max(int(nbytes.value), 1), dtype=torch.uint8, device=dev)
        self.sizes = torch.zeros(5 * L, dtype=torch.int64, device=dev)

    def launch(self, d_qoff, d_qverts, seed, epoch, batch_offset, stream=None):
        L = len(self.fanouts)
        _lib.check(_lib.lib().gb_ladies_bulk(
            self.dg.handle, self.k, _lib.ptr(d_qoff), _lib.ptr(d_qverts), self.q1_cap, L,
            self.h_fanouts.ctypes.data, int(seed), int(epoch), int(batch_offset),
            LADIES_MODES[self.mode], self.c_layers, _lib.ptr(self.sizes), _lib.ptr(self.ws),
            self.ws.numel(), _lib.stream_ptr(stream)), "gb_ladies_bulk")

    def layers(self, d_qoff, d_qverts, sizes=None):
        if sizes is None:
            sizes = self.sizes.cpu().numpy()
        if len(sizes) and sizes[-1] < 0:
            code = -int(sizes[-1])
            if code & 2:
                raise ContractViolation("LADIES batch with more than 65535 vertices: counts "
                                        "are kept in 16-bit counters")
            raise RuntimeError(f"LADIES bulk capacity overflow (code {code}: race tie list)")
        n = self.dg.n
        out = []
        qoff, qcol = d_qoff, d_qverts
        for l in range(len(self.fanouts)):
            QN, F, A, C = (int(x) for x in sizes[5 * l: 5 * l + 4])
            o = self.out[l]
            dev = {
                "frontier_shape": (self.k, n), "frontier_ptr": o["fptr"],
                "frontier_col": o["fcol"][:F],
                "adj_shape": (QN, C), "adj_ptr": o["aptr"][: QN + 1], "adj_col": o["acol"][:A],
                "rowv_off": qoff, "rowv_cat": qcol[:QN],
                "colv_off": o["fptr"], "colv_cat": o["fcol"][:F],
                "sampv_off": o["fptr"], "sampv_cat": o["fcol"][:F],
            }
            out.append(LayerSample(l + 1, device=dev, n=n))
            qoff, qcol = o["fptr"], o["fcol"]
        return out


def ladies_epoch(G, cfg, batches, epoch, batch_offset, mode="auto"):
    dg = G.device()
    d_off, d_cat, q1 = upload_batches(batches, G.n, sort_within=True)
    if mode == "auto":
        mode = "exact" if G.n * max(cfg.fanouts) <= LADIES_EXACT_LIMIT else "race"
    bulk = LadiesBulk(dg, len(batches), max(q1, 1), cfg.fanouts, mode=mode)
    bulk.launch(d_off, d_cat, cfg.seed, epoch, batch_offset)
    layers = bulk.layers(d_off, d_cat)
    return SampledEpoch(SamplerKind.LADIES, epoch, batches, layers, cfg.layers)


def sample_epoch_generic(G, cfg, batches, epoch, batch_offset, prob_spgemm):
    """sample_epoch_bulk with a user `prob_spgemm(Q) -> P` hook (reference
    sampler.py:337-345, 360-379): P is materialised by the hook, then
    normalised, sampled and extracted by the generic device operators."""
    from . import ops
    from . import sampler as smp

    n = G.n
    batch_ids = [batch_offset + i for i in range(len(batches))]
    if cfg.kind is SamplerKind.SAGE:
        Q = smp.sage_seed_matrix(batches, n)
        rows_actual = [len(b) for b in batches]
        row_vertices = [np.asarray(b).copy() for b in batches]
    else:
        Q = smp.ladies_seed_matrix(batches, n)
        rows_actual = [1] * len(batches)
        row_vertices = [np.sort(b) for b in batches]
    layers = []
    calls = 0
    for depth in range(1, cfg.layers + 1):
        fanout = cfg.fanouts[depth - 1]
        P = prob_spgemm(Q)
        calls += 1
        P = ops.norm_rows_sage(P) if cfg.kind is SamplerKind.SAGE else ops.norm_rows_ladies(P)
        keys = smp.global_row_keys(cfg, depth, batch_ids, rows_actual)
        ordered = ops.sample_rows_ordered(P, fanout, epoch, depth, cfg.seed, keys)
        frontier = ops.frontier_from_rows(ordered, P.n_cols)
        row_starts = np.cumsum([0] + rows_actual)
        if cfg.kind is SamplerKind.SAGE:
            blocks, col_maps, new_rows = smp.sage_batch_blocks(frontier, row_starts)
            layers.append(smp.build_sage_layer(depth, frontier, blocks, col_maps, row_vertices,
                                               new_rows))
            Q = ops.expand_row_extraction(frontier)
            rows_actual = [len(v) for v in new_rows]
            row_vertices = new_rows
        else:
            QR = ops.expand_row_extraction(Q)
            AR = ops.spgemm(QR, G.host_adjacency())
            ar, qc, sampled = smp.ladies_batch_blocks(Q, frontier, AR, n)
            adjacency = smp.ladies_assemble(ar, qc)
            layers.append(smp.build_ladies_layer(depth, frontier, adjacency, row_vertices,
                                                 sampled))
            Q = frontier
            row_vertices = sampled
    return SampledEpoch(cfg.kind, epoch, batches, layers, calls)


class _PinnedBlock:
    """One bulk's host results: a pinned byte tensor of the sampler's pool.
    numpy arrays made from it keep it alive (it is their base); when the last
    one is gone the tensor returns to the pool for a later bulk."""

    def __init__(self, tensor, pool):
        self.t, self.pool = tensor, pool
        self.__array_interface__ = {"shape": (tensor.numel(),), "typestr": "|u1",
                                    "data": (tensor.data_ptr(), False), "version": 3}

    def __del__(self):
        try:
            self.pool.append(self.t)
        except Exception:
            pass


class BulkSampler:
    """Public reusable bulk sampler bound to (graph, config).

    `sample(batches)` is the drop-in for `sample_epoch_bulk` when the same
    shapes recur (an epoch loop): device buffers are planned once, host
    batches travel through pinned memory, and with `to_host=True` the result
    arrays come back into pinned host memory owned by the returned epoch
    (the reference returns new host numpy arrays; here the reference types —
    `frontier` / `adjacency` SparseMatrix, the per-batch vertex tuples — are
    zero-copy views of them).  With `to_host=False` the results stay in HBM.
    SAGE (any kernel mode) and LADIES (race / exact).
    """

    def __init__(self, G: Graph, cfg: SamplerConfig, max_batch_vertices=None, mode=None):
        import torch

        self.G, self.cfg = G, cfg
        self.kind = cfg.kind
        if mode is None:
            mode = "dedup" if cfg.kind is SamplerKind.SAGE else "race"
        self.mode = mode
        self.dg = G.device()
        self.r1 = int(max_batch_vertices or cfg.bulk_count * cfg.batch_size)
        self._slots = [self._new_slot()]
        self._pool = []  # pinned result blocks not owned by a live epoch
        self._copy_stream = torch.cuda.Stream()
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def _new_slot(self):
        """Device buffers + pinned input staging of one in-flight bulk."""
        import torch

        k, r1, cfg = self.cfg.bulk_count, self.r1, self.cfg
        if self.kind is SamplerKind.SAGE:
            bulk = SageBulk(self.dg, k, r1, cfg.batch_size, cfg.fanouts, mode=self.mode)
            nsz = 3 * cfg.layers
        else:
            bulk = LadiesBulk(self.dg, k, r1, cfg.fanouts, mode=self.mode)
            nsz = 5 * cfg.layers
        return {
            "bulk": bulk,
            "h_off": torch.empty(k + 1, dtype=torch.int64, pin_memory=True),
            "h_cat": torch.empty(max(r1, 1), dtype=torch.int32, pin_memory=True),
            "d_off": torch.empty(k + 1, dtype=torch.int64, device="cuda"),
            "d_cat": torch.empty(max(r1, 1), dtype=torch.int32, device="cuda"),
            "h_sizes": torch.empty(nsz, dtype=torch.int64, pin_memory=True),
            "copied": None,
        }

    @property
    def bulk(self):
        return self._slots[0]["bulk"]

    def _upload(self, slot, batches):
        k = self.cfg.bulk_count
        if len(batches) != k:
            raise ContractViolation(f"BulkSampler built for {k} batches, got {len(batches)}")
        sort_within = self.kind is SamplerKind.LADIES
        cat, off = _flatten_batches(batches, self.G.n, sort_within=sort_within)
        if k and self.kind is SamplerKind.SAGE and \
                int(np.max(np.diff(off))) > self.cfg.batch_size:
            raise ContractViolation("actual rows exceed the nominal stride")
        if cat.size > slot["h_cat"].numel():
            raise ContractViolation("more batch vertices than the sampler was built for")
        r1 = int(off[-1])
        slot["h_off"].numpy()[:] = off
        slot["h_cat"].numpy()[:r1] = cat
        slot["d_off"].copy_(slot["h_off"], non_blocking=True)
        slot["d_cat"][:r1].copy_(slot["h_cat"][:r1], non_blocking=True)
        self.h2d_bytes = 8 * (k + 1) + 4 * r1
        return cat, off

    def _launch(self, slot, epoch, batch_offset):
        slot["bulk"].launch(slot["d_off"], slot["d_cat"], self.cfg.seed, epoch, batch_offset)
        slot["h_sizes"].copy_(slot["bulk"].sizes, non_blocking=True)

    def _stage(self, slot, layers):
        """One device->host copy per distinct device buffer, into one pinned
        block from the sampler's pool (the epoch built on it owns it until
        its last array is dropped, then it returns to the pool).  Offset
        arrays travel as int32 (values < 2^31), halving their bytes; the
        frontier, adjacency, sampled-vertex and next-layer row arrays alias
        each other and cross once."""
        import torch

        plan, seen, off = [], set(), 0
        for layer in layers:
            for key, v in layer.device.items():
                if isinstance(v, tuple):
                    continue
                ident = (v.data_ptr(), v.numel())
                if ident in seen or v.data_ptr() in (slot["d_off"].data_ptr(),
                                                     slot["d_cat"].data_ptr()):
                    continue
                seen.add(ident)
                src = v.to(torch.int32) if v.dtype == torch.int64 else v
                nb = src.numel() * src.element_size()
                plan.append((ident, src, off))
                off += (nb + 255) & ~255
        need = max(off, 256)
        blk = None
        for i, t in enumerate(self._pool):
            if t.numel() >= need:
                blk = self._pool.pop(i)
                break
        if blk is None:
            blk = torch.empty(need + need // 8, dtype=torch.uint8, pin_memory=True)
        host = {}
        nbytes = 0
        for ident, src, o in plan:
            n = src.numel() * src.element_size()
            if n:
                blk[o:o + n].view(src.dtype).copy_(src, non_blocking=True)
            host[ident] = (o, src.dtype, src.numel())
            nbytes += n
        return (_PinnedBlock(blk, self._pool), host), nbytes

    def _host_epoch(self, slot, layers, staged, batches, cat, off, epoch):
        import torch

        block, host = staged
        base = np.asarray(block)  # keeps the block (and its pool slot) alive
        np_dtype = {torch.int32: np.int32, torch.int64: np.int64, torch.float32: np.float32}
        out_layers = []
        for layer in layers:
            h = {}
            for key, v in layer.device.items():
                if isinstance(v, tuple):
                    h[key] = np.asarray(v, dtype=np.int64)
                elif v.data_ptr() == slot["d_off"].data_ptr():
                    h[key] = off
                elif v.data_ptr() == slot["d_cat"].data_ptr():
                    h[key] = cat[: v.numel()]
                else:
                    o, dt, n = host[(v.data_ptr(), v.numel())]
                    item = np.dtype(np_dtype[dt]).itemsize
                    h[key] = base[o:o + n * item].view(np_dtype[dt])
            out_layers.append(LayerSample(layer.depth, device=h, n=self.G.n))
        return SampledEpoch(self.kind, epoch, batches, out_layers, self.cfg.layers)

    def _layers(self, slot, sizes):
        return slot["bulk"].layers(slot["d_off"], slot["d_cat"], sizes)

    def sample(self, batches, epoch=0, batch_offset=0, to_host=True) -> SampledEpoch:
        import torch

        slot = self._slots[0]
        if slot["copied"] is not None:
            slot["copied"].synchronize()
        cat, off = self._upload(slot, batches)
        self._launch(slot, epoch, batch_offset)
        torch.cuda.current_stream().synchronize()
        sizes = slot["h_sizes"].numpy().copy()
        layers = self._layers(slot, sizes)
        self.d2h_bytes = 8 * sizes.size
        if not to_host:
            return SampledEpoch(self.kind, epoch, batches, layers, self.cfg.layers)
        host, nbytes = self._stage(slot, layers)
        self.d2h_bytes += nbytes
        torch.cuda.current_stream().synchronize()
        return self._host_epoch(slot, layers, host, batches, cat, off, epoch)

    def sample_stream(self, jobs, epoch=0):
        """Generator over `jobs` (an iterable of (batches, batch_offset)):
        yields each bulk's host SampledEpoch, with the device->host copy of
        bulk j (side stream) overlapping the sampling of bulk j + 1 (two
        device buffer sets alternate).  Same results as sample(); every
        yielded epoch owns its host memory.
        """
        import torch

        if len(self._slots) < 2:
            self._slots.append(self._new_slot())
        cs = torch.cuda.current_stream()
        xs = self._copy_stream
        pend = None
        j = 0
        for batches, boff in jobs:
            slot = self._slots[j % 2]
            if slot["copied"] is not None:
                cs.wait_event(slot["copied"])  # its previous bulk left the device
                slot["copied"].synchronize()   # and its pinned inputs are free
            cat, off = self._upload(slot, batches)
            self._launch(slot, epoch, boff)
            done = torch.cuda.Event()
            done.record(cs)
            done.synchronize()  # sizes of bulk j (bulk j - 1 is still copying)
            sizes = slot["h_sizes"].numpy().copy()
            layers = self._layers(slot, sizes)
            xs.wait_event(done)
            with torch.cuda.stream(xs):
                host, nbytes = self._stage(slot, layers)
            slot["copied"] = torch.cuda.Event()
            slot["copied"].record(xs)
            self.d2h_bytes = 8 * sizes.size + nbytes
            if pend is not None:
                pslot, pev, players, phost, pb, pcat, poff = pend
                pev.synchronize()
                yield self._host_epoch(pslot, players, phost, pb, pcat, poff, epoch)
            pend = (slot, slot["copied"], layers, host, batches, cat, off)
            j += 1
        if pend is not None:
            pslot, pev, players, phost, pb, pcat, poff = pend
            pev.synchronize()
            yield self._host_epoch(pslot, players, phost, pb, pcat, poff, epoch)
