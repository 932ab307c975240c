"""Synthetic OGB-shaped graphs built on the device (SURVEY.md §8(d) inputs).

Canonical recipe: Graph500 R-MAT (a, b, c) =
(0.57, 0.19, 0.19) over scale = ceil(log2 n) levels, reject ids >= n and self
loops, keep the first m distinct (undirected) pairs in draw order, random
relabel, symmetrise (papers shape stays directed), sorted de-duplicated CSR.
Everything runs in the library (`gb_rmat_graph`: Philox-keyed candidates,
radix sorts, scans); `oracle/csrc/gen.c` builds the identical CSR on the host.

Difference from the host recipe: draws come from Philox keyed by the draw
index (parallel, identical on every device) instead of one sequential
PCG64 stream, and the relabelling permutation is the rank of a keyed hash.
"""

from __future__ import annotations

from . import _lib
from .sparse import DeviceGraph, Graph

SHAPES = {
    # name: (n, m, symmetric) — BASELINE.md §2 table
    "cfg1": (65_536, 1_048_576, True),
    "products": (2_449_029, 61_859_140, True),
    "papers": (111_059_956, 1_615_685_872, False),
}


def rmat_device_graph(n, m, symmetric=True, seed=0, a=0.57, b=0.19, c=0.19) -> DeviceGraph:
    """R-MAT graph with exactly m distinct pairs (2m directed entries when
    symmetric), built on the current CUDA device."""
    import ctypes

    import torch

    n, m = int(n), int(m)
    E = 2 * m if symmetric else m
    L = _lib.lib()
    cand = int(m * 1.3) + 4096
    rowptr = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(E + _lib.GB_COL_PAD, dtype=torch.int32, device="cuda")
    info = (ctypes.c_int64 * 2)()
    while True:
        nbytes = L.gb_rmat_graph_workspace(n, m, int(bool(symmetric)), cand)
        ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device="cuda")
        rc = L.gb_rmat_graph(seed, n, m, int(bool(symmetric)), a, b, c, cand, _lib.ptr(rowptr),
                             _lib.ptr(col), col.numel(), info, _lib.ptr(ws), ws.numel(),
                             _lib.stream_ptr())
        del ws
        if rc == _lib.GB_ERR_CAPACITY and info[1] < m:
            # too few distinct pairs among the candidates: draw more
            cand = int(cand * m / max(int(info[1]), 1) * 1.05) + 4096
            continue
        _lib.check(rc, "gb_rmat_graph")
        break
    torch.cuda.synchronize()
    return DeviceGraph(n, rowptr, col, int(info[0]))


def rmat_device_block(n, m, symmetric, row_lo, row_hi, seed=0, a=0.57, b=0.19, c=0.19):
    """Rows [row_lo, row_hi) of rmat_device_graph(n, m, symmetric, seed) as a
    block CSR (local rows, global columns; gb_rmat_block): (rowptr int64,
    col int32 padded by GB_COL_PAD, nnz)."""
    import ctypes

    import torch

    n, m, lo, hi = int(n), int(m), int(row_lo), int(row_hi)
    E = 2 * m if symmetric else m
    L = _lib.lib()
    cand = int(m * 1.3) + 4096
    cap = int(E * (hi - lo) / n * 1.25) + (1 << 16)
    info = (ctypes.c_int64 * 2)()
    rowptr = torch.empty(hi - lo + 1, dtype=torch.int64, device="cuda")
    while True:
        col = torch.empty(cap + _lib.GB_COL_PAD, dtype=torch.int32, device="cuda")
        nbytes = L.gb_rmat_graph_workspace(n, m, int(bool(symmetric)), cand)
        ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device="cuda")
        rc = L.gb_rmat_block(seed, n, m, int(bool(symmetric)), a, b, c, cand, lo, hi,
                             _lib.ptr(rowptr), _lib.ptr(col), col.numel(), info, _lib.ptr(ws),
                             ws.numel(), _lib.stream_ptr())
        del ws
        if rc == _lib.GB_ERR_CAPACITY and info[1] < m:
            cand = int(cand * m / max(int(info[1]), 1) * 1.05) + 4096
            continue
        if rc == _lib.GB_ERR_CAPACITY and info[0] > cap:
            cap = int(info[0])
            continue
        _lib.check(rc, "gb_rmat_block")
        break
    nnz = int(info[0])
    if col.numel() > nnz + _lib.GB_COL_PAD + (1 << 20):  # trim the estimate
        col = col[: nnz + _lib.GB_COL_PAD].clone()
    torch.cuda.synchronize()
    return rowptr, col, nnz


def synthetic_graph(shape="products", seed=0) -> Graph:
    n, m, sym = SHAPES[shape]
    return Graph.from_device(rmat_device_graph(n, m, symmetric=sym, seed=seed))
