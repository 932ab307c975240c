"""Synthetic OGB-shaped graphs built on the device (SURVEY.md §8(d) inputs).

Canonical recipe: Graph500 R-MAT (a, b, c) =
(0.57, 0.19, 0.19) over scale = ceil(log2 n) levels, reject ids >= n and self
loops, keep m unique (undirected) pairs, random relabel, symmetrise
(papers shape stays directed), sorted de-duplicated CSR.  Candidates come
from the library's Philox-driven R-MAT kernel (gb_rmat_edges) and the
relabelling from its keyed hash (gb_hash64), so every device produces the
same graph; sorting/de-duplication uses torch on the device (plumbing).

Difference from the host recipe: when more than m unique pairs were drawn,
the m kept are the ones with the smallest keyed hash (a deterministic
uniform subset) instead of the first m in draw order.
"""

from __future__ import annotations

import math

from . import _lib
from .sparse import DeviceGraph, Graph

SHAPES = {
    # name: (n, m, symmetric) — BASELINE.md §2 table
    "cfg1": (65_536, 1_048_576, True),
    "products": (2_449_029, 61_859_140, True),
    "papers": (111_059_956, 1_615_685_872, False),
}


def _rmat_candidates(seed, scale, n, first, count, a, b, c):
    import torch

    src = torch.empty(count, dtype=torch.int64, device="cuda")
    dst = torch.empty(count, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().gb_rmat_edges(seed, scale, n, first, count, a, b, c, _lib.ptr(src),
                                        _lib.ptr(dst), _lib.stream_ptr()), "gb_rmat_edges")
    return src, dst


def _hash(seed, x):
    import torch

    out = torch.empty_like(x)
    _lib.check(_lib.lib().gb_hash64(seed, _lib.ptr(x), x.numel(), _lib.ptr(out),
                                    _lib.stream_ptr()), "gb_hash64")
    return out


def rmat_device_graph(n, m, symmetric=True, seed=0, a=0.57, b=0.19, c=0.19) -> DeviceGraph:
    """R-MAT graph with exactly m unique pairs (2m directed entries when
    symmetric), entirely on the current CUDA device."""
    import torch

    n, m = int(n), int(m)
    scale = max(1, math.ceil(math.log2(n)))
    keys = torch.empty(0, dtype=torch.int64, device="cuda")
    first = 0
    while keys.numel() < m:
        need = m - keys.numel()
        count = int(need * 1.35) + 4096
        src, dst = _rmat_candidates(seed, scale, n, first, count, a, b, c)
        first += count
        ok = src >= 0
        src, dst = src[ok], dst[ok]
        if symmetric:
            src, dst = torch.minimum(src, dst), torch.maximum(src, dst)
        new = src * n + dst
        del src, dst, ok
        keys = torch.unique(torch.cat([keys, new]))
        del new
    if keys.numel() > m:
        order = torch.argsort(_hash(seed + 1, keys))[:m]
        keys = keys[order]
        del order
    # random relabel: label[v] = rank of hash(v)
    ids = torch.arange(n, dtype=torch.int64, device="cuda")
    perm = torch.argsort(_hash(seed + 2, ids))
    label = torch.empty_like(perm)
    label[perm] = ids
    del perm, ids
    u = label[keys // n]
    v = label[keys % n]
    del keys, label
    if symmetric:
        u, v = torch.cat([u, v]), torch.cat([v, u])
    key = torch.sort(u * n + v).values
    del u, v
    src = key // n
    rowptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    rowptr[1:] = torch.cumsum(torch.bincount(src, minlength=n), 0)
    del src
    nnz = key.numel()
    col = torch.zeros(nnz + _lib.GB_COL_PAD, dtype=torch.int32, device="cuda")
    col[:nnz] = (key % n).to(torch.int32)
    del key
    torch.cuda.synchronize()
    return DeviceGraph(n, rowptr, col, nnz)


def synthetic_graph(shape="products", seed=0) -> Graph:
    n, m, sym = SHAPES[shape]
    return Graph.from_device(rmat_device_graph(n, m, symmetric=sym, seed=seed))
