"""Device implementations of the reference's sparse / sampling operators.

Same names, argument meaning and errors as `pkg/src/gnnbulk/sparse.py` and
`sampler.py`; inputs and outputs are the host `SparseMatrix` type (the
compatibility edge) and every compute step runs on the GPU:

* `spgemm`, `add`, `norm_rows_sage`, `norm_rows_ladies`, the ITS samplers:
  hand-written kernels in csrc/gb_ops.cu (bit-exact with scipy / numpy
  orders, see that file);
* the structural helpers (vstack, block_diag, compact_columns,
  expand_row_extraction, column_window, rows_subset,
  build_column_extraction, frontier_from_rows) are index manipulations
  done with device tensor primitives.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ContractViolation
from .sparse import SparseMatrix


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2311_02909_b200 ops need a CUDA device; no CPU fallback")
    return torch


class DeviceCSR:
    """CSR in HBM: ptr int64[n_rows+1], col int32[nnz], val float64[nnz]."""

    __slots__ = ("n_rows", "n_cols", "ptr", "col", "val")

    def __init__(self, n_rows, n_cols, ptr, col, val):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.ptr, self.col, self.val = ptr, col, val

    @property
    def nnz(self):
        return int(self.col.numel())

    @classmethod
    def from_host(cls, M: SparseMatrix):
        torch = _torch()
        if M.n_cols >= 2**31:
            raise ContractViolation("column count must be < 2^31 on the device")
        return cls(M.n_rows, M.n_cols,
                   torch.as_tensor(np.array(M.row_offsets, dtype=np.int64)).cuda(),
                   torch.as_tensor(np.array(M.col_indices, dtype=np.int32)).cuda(),
                   torch.as_tensor(np.array(M.values, dtype=np.float64)).cuda())

    def to_host(self) -> SparseMatrix:
        return SparseMatrix(self.n_rows, self.n_cols, self.ptr.cpu().numpy(),
                            self.col.cpu().numpy().astype(np.int64), self.val.cpu().numpy(),
                            validate=False)


def _dev(M):
    return M if isinstance(M, DeviceCSR) else DeviceCSR.from_host(M)


def _scalar(x):
    torch = _torch()
    return torch.tensor([int(x)], dtype=torch.int64, device="cuda")


def _scan_ws(n):
    torch = _torch()
    nbytes = _lib.lib().gb_scan_workspace_bytes(int(n))
    return torch.empty(max(nbytes // 8, 1), dtype=torch.int64, device="cuda")


# -- RNG -------------------------------------------------------------------------


def uniforms(seed, epoch, depth, rows, t):
    """u(seed, epoch, depth, row, t) on the device (gb_uniforms)."""
    torch = _torch()
    rows = torch.as_tensor(np.asarray(rows, dtype=np.int64)).cuda()
    t = torch.as_tensor(np.asarray(t, dtype=np.int64)).cuda()
    out = torch.empty(rows.numel(), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().gb_uniforms(int(seed), int(epoch), int(depth), _lib.ptr(rows),
                                      _lib.ptr(t), rows.numel(), _lib.ptr(out),
                                      _lib.stream_ptr()), "gb_uniforms")
    return out.cpu().numpy()


# -- kernels -------------------------------------------------------------------------


def spgemm_device(A: DeviceCSR, B: DeviceCSR) -> DeviceCSR:
    torch = _torch()
    m = A.n_rows
    d_m = _scalar(m)
    ws = _scan_ws(m)
    ub = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    L = _lib.lib()
    _lib.check(L.gb_spgemm_bound(m, _lib.ptr(A.ptr), _lib.ptr(A.col), _lib.ptr(B.ptr),
                                 _lib.ptr(d_m), _lib.ptr(ub), _lib.ptr(ws), _lib.stream_ptr()),
               "gb_spgemm_bound")
    total = int(ub[m].item())
    cap = max(total, 1)
    gkey = torch.empty(4 * cap, dtype=torch.int32, device="cuda")
    gval = torch.empty(4 * cap, dtype=torch.float64, device="cuda")
    tcol = torch.empty(cap, dtype=torch.int32, device="cuda")
    tval = torch.empty(cap, dtype=torch.float64, device="cuda")
    cnt = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    cptr = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    ccol = torch.empty(cap, dtype=torch.int32, device="cuda")
    cval = torch.empty(cap, dtype=torch.float64, device="cuda")
    _lib.check(L.gb_spgemm(m, _lib.ptr(d_m), _lib.ptr(A.ptr), _lib.ptr(A.col), _lib.ptr(A.val),
                           _lib.ptr(B.ptr), _lib.ptr(B.col), _lib.ptr(B.val), _lib.ptr(ub), total,
                           _lib.ptr(gkey), _lib.ptr(gval), _lib.ptr(tcol), _lib.ptr(tval),
                           _lib.ptr(cnt), _lib.ptr(cptr), _lib.ptr(ccol), _lib.ptr(cval),
                           _lib.ptr(ws), _lib.stream_ptr()), "gb_spgemm")
    nnz = int(cptr[m].item())
    return DeviceCSR(m, B.n_cols, cptr, ccol[:nnz], cval[:nnz])


def spgemm(left: SparseMatrix, right: SparseMatrix) -> SparseMatrix:
    """left @ right with the reference's drop policy (sparse.py:233-251)."""
    if left.n_cols != right.n_rows:
        raise ContractViolation(f"spgemm dimension mismatch: {left.shape} @ {right.shape}")
    return spgemm_device(_dev(left), _dev(right)).to_host()


def add_device(A: DeviceCSR, B: DeviceCSR) -> DeviceCSR:
    torch = _torch()
    m = A.n_rows
    d_m = _scalar(m)
    ws = _scan_ws(m)
    cnt = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    cptr = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    L = _lib.lib()
    args = [m, _lib.ptr(d_m), _lib.ptr(A.ptr), _lib.ptr(A.col), _lib.ptr(A.val), _lib.ptr(B.ptr),
            _lib.ptr(B.col), _lib.ptr(B.val), _lib.ptr(cnt), _lib.ptr(cptr)]
    _lib.check(L.gb_csr_add(*args, _lib.ptr(None), _lib.ptr(None), _lib.ptr(ws), 0,
                            _lib.stream_ptr()), "gb_csr_add")
    nnz = int(cptr[m].item())
    ccol = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
    cval = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
    _lib.check(L.gb_csr_add(*args, _lib.ptr(ccol), _lib.ptr(cval), _lib.ptr(ws), 1,
                            _lib.stream_ptr()), "gb_csr_add")
    return DeviceCSR(m, A.n_cols, cptr, ccol[:nnz], cval[:nnz])


def add(left: SparseMatrix, right: SparseMatrix) -> SparseMatrix:
    """Elementwise sum, cancellation below 1e-12 dropped (sparse.py:417-427)."""
    if left.shape != right.shape:
        raise ContractViolation(f"add shape mismatch: {left.shape} vs {right.shape}")
    return add_device(_dev(left), _dev(right)).to_host()


def _norm(P, square):
    torch = _torch()
    D = _dev(P)
    if D.nnz == 0:
        return P if isinstance(P, SparseMatrix) else D
    out = torch.empty_like(D.val)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().gb_norm_rows(D.n_rows, _lib.ptr(D.ptr), _lib.ptr(D.val), int(square),
                                       _lib.ptr(out), _lib.ptr(err), _lib.stream_ptr()),
               "gb_norm_rows")
    e = int(err.item())
    if e == 1:
        raise ContractViolation("row normalization requires non-negative values")
    if e == 2:
        raise ContractViolation("nonempty row with zero mass cannot be normalized")
    res = DeviceCSR(D.n_rows, D.n_cols, D.ptr, D.col, out)
    return res.to_host() if isinstance(P, SparseMatrix) else res


def norm_rows_sage(P):
    """v / row sum (sparse.py:254-260)."""
    return _norm(P, False)


def norm_rows_ladies(P):
    """e^2 / row sum of squares (sparse.py:263-269)."""
    return _norm(P, True)


def _its(D: DeviceCSR, s, keys=None, inject=None, seed=0, epoch=0, depth=0):
    torch = _torch()
    m = D.n_rows
    nnz = max(D.nnz, 1)
    w = torch.empty(nnz, dtype=torch.float64, device="cuda")
    cdf = torch.empty(nnz, dtype=torch.float64, device="cuda")
    picks = torch.full((max(m * s, 1),), -1, dtype=torch.int32, device="cuda")
    take = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().gb_its_rows(m, _lib.ptr(D.ptr), _lib.ptr(D.val), int(s),
                                      _lib.ptr(keys), _lib.ptr(inject), int(seed), int(epoch),
                                      int(depth), _lib.ptr(w), _lib.ptr(cdf), _lib.ptr(picks),
                                      _lib.ptr(take), _lib.ptr(err), _lib.stream_ptr()),
               "gb_its_rows")
    if int(err.item()):
        raise ContractViolation("probabilities must be positive")
    return picks.view(-1)[: m * s].view(m, s) if m else picks[:0].view(0, s), take[:m]


def its_sample_row(probabilities, s, rng) -> np.ndarray:
    """min(s, m) distinct indices in draw order (sampler.py:157-189); the
    uniforms are `rng.random()` draws (t-th draw for the t-th pick)."""
    torch = _torch()
    w = np.asarray(probabilities, dtype=np.float64)
    m = w.size
    if m == 0:
        return np.zeros(0, dtype=np.int64)
    if w.min() <= 0:
        raise ContractViolation("probabilities must be positive")
    take = min(int(s), m)
    us = np.zeros(int(s), dtype=np.float64)
    if take < m:
        for t in range(take):
            us[t] = rng.random()
    D = DeviceCSR(1, m, torch.tensor([0, m], dtype=torch.int64, device="cuda"),
                  torch.arange(m, dtype=torch.int32, device="cuda"),
                  torch.as_tensor(w).cuda())
    picks, tk = _its(D, int(s), inject=torch.as_tensor(us).cuda())
    return picks[0, : int(tk[0].item())].cpu().numpy().astype(np.int64)


def sample_rows_ordered(P, s, epoch, layer, seed, row_keys=None):
    """Sampled column ids of every row, in draw order (sampler.py:192-207)."""
    torch = _torch()
    D = _dev(P)
    keys = np.arange(D.n_rows, dtype=np.int64) if row_keys is None else np.asarray(
        row_keys, dtype=np.int64)
    picks, take = _its(D, int(s), keys=torch.as_tensor(keys).cuda(), seed=seed, epoch=epoch,
                       depth=layer)
    ptr = D.ptr.cpu().numpy()
    col = D.col.cpu().numpy().astype(np.int64)
    pk = picks.cpu().numpy()
    tk = take.cpu().numpy()
    return [col[ptr[r] + pk[r, : tk[r]]] for r in range(D.n_rows)]


def frontier_from_rows(sampled_rows, n_cols) -> SparseMatrix:
    """Value-1 frontier matrix with row r = sorted sampled_rows[r] (sampler.py:210-222)."""
    torch = _torch()
    lens = np.array([len(x) for x in sampled_rows], dtype=np.int64)
    ptr = np.zeros(len(sampled_rows) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(lens)
    cat = np.concatenate([np.asarray(x, dtype=np.int64) for x in sampled_rows]) if len(
        sampled_rows) else np.zeros(0, np.int64)
    rows = torch.repeat_interleave(torch.arange(len(sampled_rows), device="cuda"),
                                   torch.as_tensor(lens).cuda())
    key = rows * max(int(n_cols), 1) + torch.as_tensor(cat).cuda()
    srt = torch.sort(key).values
    col = (srt % max(int(n_cols), 1)).cpu().numpy()
    return SparseMatrix(len(sampled_rows), n_cols, ptr, col, np.ones(col.size), validate=False)


def sample_frontier(P, s, epoch, layer, seed, row_keys=None) -> SparseMatrix:
    """min(s, nnz) sampled columns per row as a value-1 matrix (sampler.py:225-234)."""
    return frontier_from_rows(sample_rows_ordered(P, s, epoch, layer, seed, row_keys), P.n_cols)


# -- structural helpers (sparse.py:289-446) ----------------------------------------


def vstack(blocks, n_cols=None) -> SparseMatrix:
    blocks = list(blocks)
    if not blocks:
        if n_cols is None:
            raise ContractViolation("vstack of an empty list requires n_cols")
        return SparseMatrix.empty(0, n_cols)
    width = blocks[0].n_cols
    if n_cols is not None and n_cols != width:
        raise ContractViolation("explicit n_cols disagrees with block width")
    if any(b.n_cols != width for b in blocks[1:]):
        raise ContractViolation("vstack blocks must share n_cols")
    return _stack(blocks, width, diag=False)


def block_diag(blocks) -> SparseMatrix:
    blocks = list(blocks)
    if not blocks:
        return SparseMatrix.empty(0, 0)
    return _stack(blocks, sum(b.n_cols for b in blocks), diag=True)


def _stack(blocks, width, diag):
    torch = _torch()
    ptrs, cols, vals = [np.zeros(1, np.int64)], [], []
    base, cbase = 0, 0
    for b in blocks:
        ptrs.append(np.asarray(b.row_offsets[1:], np.int64) + base)
        c = torch.as_tensor(np.array(b.col_indices, np.int64)).cuda()
        cols.append(c + cbase if diag else c)
        vals.append(np.asarray(b.values))
        base += b.nnz
        cbase += b.n_cols
    col = torch.cat(cols).cpu().numpy() if cols else np.zeros(0, np.int64)
    return SparseMatrix(sum(b.n_rows for b in blocks), width, np.concatenate(ptrs), col,
                        np.concatenate(vals), validate=False)


def compact_columns(M: SparseMatrix):
    """Drop empty columns; returns (compacted, column_map) (sparse.py:345-357)."""
    torch = _torch()
    c = torch.as_tensor(np.array(M.col_indices, np.int64)).cuda()
    kept = torch.unique(c)
    new = torch.searchsorted(kept, c)
    out = SparseMatrix(M.n_rows, int(kept.numel()), M.row_offsets, new.cpu().numpy(), M.values,
                       validate=False)
    return out, kept.cpu().numpy()


def expand_row_extraction(Q: SparseMatrix) -> SparseMatrix:
    """One one-hot row per nonzero of Q, in order (sparse.py:360-370)."""
    m = Q.nnz
    return SparseMatrix(m, Q.n_cols, np.arange(m + 1), Q.col_indices, np.ones(m), validate=False)


def column_window(M: SparseMatrix, lo: int, hi: int) -> SparseMatrix:
    """Entries with column in [lo, hi), shifted to 0 (sparse.py:373-388)."""
    torch = _torch()
    if not (0 <= lo <= hi <= M.n_cols):
        raise ContractViolation(f"column window [{lo}, {hi}) out of range")
    c = torch.as_tensor(np.array(M.col_indices, np.int64)).cuda()
    ptr = torch.as_tensor(np.array(M.row_offsets, np.int64)).cuda()
    keep = (c >= lo) & (c < hi)
    rows = torch.repeat_interleave(torch.arange(M.n_rows, device="cuda"), ptr[1:] - ptr[:-1])
    counts = torch.bincount(rows[keep], minlength=M.n_rows)
    nptr = torch.zeros(M.n_rows + 1, dtype=torch.int64, device="cuda")
    nptr[1:] = torch.cumsum(counts, 0)
    kk = keep.cpu().numpy()
    return SparseMatrix(M.n_rows, hi - lo, nptr.cpu().numpy(), (c[keep] - lo).cpu().numpy(),
                        np.asarray(M.values)[kk], validate=False)


def rows_subset(M: SparseMatrix, rows) -> SparseMatrix:
    """Copy of M keeping only the given rows (sparse.py:391-414)."""
    torch = _torch()
    r = torch.unique(torch.as_tensor(np.asarray(rows, np.int64)).cuda())
    if r.numel() and (int(r[0]) < 0 or int(r[-1]) >= M.n_rows):
        raise ContractViolation("row id out of range")
    ptr = torch.as_tensor(np.array(M.row_offsets, np.int64)).cuda()
    deg = ptr[1:] - ptr[:-1]
    counts = torch.zeros(M.n_rows, dtype=torch.int64, device="cuda")
    counts[r] = deg[r]
    nptr = torch.zeros(M.n_rows + 1, dtype=torch.int64, device="cuda")
    nptr[1:] = torch.cumsum(counts, 0)
    lens = deg[r]
    starts = ptr[:-1][r]
    total = int(lens.sum().item()) if r.numel() else 0
    excl = torch.cumsum(lens, 0) - lens
    gather = torch.repeat_interleave(starts - excl, lens) + torch.arange(total, device="cuda")
    g = gather.cpu().numpy()
    return SparseMatrix(M.n_rows, M.n_cols, nptr.cpu().numpy(), np.asarray(M.col_indices)[g],
                        np.asarray(M.values)[g], validate=False)


def build_column_extraction(sampled_cols, n: int) -> SparseMatrix:
    """n x s selector, column j has its 1 at row sampled_cols[j] (sparse.py:430-446)."""
    torch = _torch()
    s = np.asarray(sampled_cols, dtype=np.int64)
    if s.size:
        if s.min() < 0 or s.max() >= n:
            raise ContractViolation("sampled vertex id out of range")
        if np.unique(s).size != s.size:
            raise ContractViolation("sampled vertex ids must be distinct")
    d = torch.as_tensor(s if s.flags.writeable else s.copy()).cuda()
    order = torch.argsort(d, stable=True)
    rows = d[order]
    ptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    ptr[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    return SparseMatrix(n, s.size, ptr.cpu().numpy(), order.cpu().numpy(), np.ones(s.size),
                        validate=False)
