"""CSR containers and the device graph.

`SparseMatrix` and `Graph` keep the reference's value semantics
(`pkg/src/gnnbulk/sparse.py:31-227`): canonical CSR with int64 offsets and
columns, float64 values, strictly increasing columns per row, frozen
arrays, bitwise `equals`.  They are the host-side *compatibility edge*: the
sampler itself runs on the device through `DeviceGraph`, which holds the
adjacency as int64 row offsets + int32 columns in HBM (values are implicit
1.0) together with the exact-replay tables built by the C ABI.

The sparse *kernels* of the reference module (spgemm, normalisation,
extraction helpers) live in `paper_2311_02909_b200.ops` and run on the GPU.
"""

from __future__ import annotations

import numpy as np

from .errors import ContractViolation

INDEX_DTYPE = np.int64
VALUE_DTYPE = np.float64


def _frozen(a, dtype):
    out = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    out.setflags(write=False)
    return out


class SparseMatrix:
    """Immutable canonical CSR matrix (reference `sparse.py:31-191`)."""

    __slots__ = ("n_rows", "n_cols", "row_offsets", "col_indices", "values")

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values, validate=True):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_offsets = _frozen(row_offsets, INDEX_DTYPE)
        self.col_indices = _frozen(col_indices, INDEX_DTYPE)
        self.values = _frozen(values, VALUE_DTYPE)
        if validate:
            self.check()

    # -- invariants (reference sparse.py:52-77) --------------------------------
    def check(self):
        if self.n_rows < 0 or self.n_cols < 0:
            raise ContractViolation("matrix dimensions must be non-negative")
        ptr, col = self.row_offsets, self.col_indices
        nnz = col.shape[0]
        if ptr.shape != (self.n_rows + 1,):
            raise ContractViolation("row_offsets must have length n_rows + 1")
        if ptr[0] != 0 or ptr[-1] != nnz:
            raise ContractViolation("row_offsets must start at 0 and end at nnz")
        if self.n_rows and np.min(np.diff(ptr)) < 0:
            raise ContractViolation("row_offsets must be non-decreasing")
        if self.values.shape[0] != nnz:
            raise ContractViolation("col_indices and values must have equal length")
        if nnz:
            if col.min() < 0 or col.max() >= self.n_cols:
                raise ContractViolation("column index out of range")
            # a non-increasing step is legal only where a new row starts
            row_of = np.repeat(np.arange(self.n_rows), np.diff(ptr))
            same_row = row_of[1:] == row_of[:-1]
            if np.any(same_row & (col[1:] <= col[:-1])):
                raise ContractViolation("column indices must be sorted and unique per row")
        if not np.isfinite(self.values).all():
            raise ContractViolation("values must be finite")

    # -- constructors -------------------------------------------------------------
    @classmethod
    def from_coo(cls, n_rows, n_cols, rows, cols, vals, dedup="sum"):
        """Triplets -> canonical CSR; duplicates summed ('sum', in input order)
        or collapsed to the first occurrence's pattern entry ('first')."""
        rows = np.asarray(rows, dtype=INDEX_DTYPE).ravel()
        cols = np.asarray(cols, dtype=INDEX_DTYPE).ravel()
        vals = np.asarray(vals, dtype=VALUE_DTYPE).ravel()
        if rows.size and (rows.min() < 0 or rows.max() >= n_rows):
            raise ContractViolation("row index out of range")
        if cols.size and (cols.min() < 0 or cols.max() >= n_cols):
            raise ContractViolation("column index out of range")
        order = np.lexsort((cols, rows)) if dedup == "first" else np.argsort(
            rows * max(int(n_cols), 1) + cols, kind="stable")
        r, c, v = rows[order], cols[order], vals[order]
        start = np.ones(r.shape[0], dtype=bool)
        start[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        seg = np.flatnonzero(start)
        if dedup == "first":
            v = v[seg]
        else:
            v = np.add.reduceat(v, seg) if seg.size else v[:0]
        r, c = r[seg], c[seg]
        ptr = np.zeros(int(n_rows) + 1, dtype=INDEX_DTYPE)
        np.cumsum(np.bincount(r, minlength=int(n_rows)), out=ptr[1:])
        return cls(n_rows, n_cols, ptr, c, v)

    @classmethod
    def from_dense(cls, array):
        a = np.asarray(array, dtype=VALUE_DTYPE)
        r, c = np.nonzero(a)
        return cls.from_coo(a.shape[0], a.shape[1], r, c, a[r, c])

    @classmethod
    def from_scipy(cls, mat, shape=None):
        csr = mat.tocsr()
        csr.sort_indices()
        n_rows, n_cols = shape if shape is not None else csr.shape
        return cls(n_rows, n_cols, csr.indptr, csr.indices, csr.data)

    @classmethod
    def trusted(cls, n_rows, n_cols, row_offsets, col_indices):
        """Zero-copy view of a canonical 0/1 CSR produced by the device sampler
        (row offsets / columns as returned, int32 or int64; values a
        read-only broadcast of 1.0).  Same values and semantics as the
        reference's arrays, no host conversion."""
        m = cls.__new__(cls)
        m.n_rows, m.n_cols = int(n_rows), int(n_cols)
        ptr = np.asarray(row_offsets).view()
        col = np.asarray(col_indices).view()
        ptr.setflags(write=False)
        col.setflags(write=False)
        m.row_offsets, m.col_indices = ptr, col
        m.values = np.broadcast_to(np.float64(1.0), (col.shape[0],))
        return m

    @classmethod
    def empty(cls, n_rows, n_cols):
        return cls(n_rows, n_cols, np.zeros(int(n_rows) + 1, dtype=INDEX_DTYPE), [], [])

    @classmethod
    def identity(cls, n):
        return cls(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    # -- accessors ------------------------------------------------------------------
    @property
    def nnz(self):
        return int(self.col_indices.shape[0])

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def row_slice(self, start, stop):
        if not (0 <= start <= stop <= self.n_rows):
            raise ContractViolation(f"row slice [{start}, {stop}) out of range")
        a, b = int(self.row_offsets[start]), int(self.row_offsets[stop])
        return SparseMatrix(stop - start, self.n_cols, self.row_offsets[start:stop + 1] - a,
                            self.col_indices[a:b], self.values[a:b], validate=False)

    def row_cols(self, r):
        return self.col_indices[self.row_offsets[r]:self.row_offsets[r + 1]]

    def row_vals(self, r):
        return self.values[self.row_offsets[r]:self.row_offsets[r + 1]]

    def row_nnz(self):
        return np.diff(self.row_offsets)

    def nonzero_cols(self):
        return np.unique(self.col_indices)

    def to_scipy(self):
        import scipy.sparse as sp

        return sp.csr_matrix((self.values, self.col_indices, self.row_offsets),
                             shape=self.shape)

    def to_dense(self):
        out = np.zeros(self.shape, dtype=VALUE_DTYPE)
        rows = np.repeat(np.arange(self.n_rows), self.row_nnz())
        out[rows, self.col_indices] = self.values
        return out

    def equals(self, other):
        return (self.shape == other.shape
                and np.array_equal(self.row_offsets, other.row_offsets)
                and np.array_equal(self.col_indices, other.col_indices)
                and np.array_equal(self.values, other.values))

    def __repr__(self):
        return f"SparseMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz})"


class Graph:
    """Unweighted graph as an n x n 0/1 adjacency (reference `sparse.py:194-227`).

    `from_edges` builds the CSR on the device (`gb_csr_from_edges`); the host
    `adjacency` SparseMatrix is materialised from the device copy on first
    access, and the device copy (`device()`) from a host adjacency on first
    use.
    """

    __slots__ = ("_adj", "n", "_dev")

    def __init__(self, adjacency: SparseMatrix):
        if adjacency.n_rows != adjacency.n_cols:
            raise ContractViolation("adjacency matrix must be square")
        if adjacency.nnz and not np.all(adjacency.values == 1.0):
            raise ContractViolation("adjacency values must all equal 1.0")
        self._adj = adjacency
        self.n = adjacency.n_rows
        self._dev = None

    @classmethod
    def from_edges(cls, n, sources, targets):
        """Edge list -> Graph, duplicates collapsed (sparse.py:211-216), the
        CSR built on the device."""
        src = np.asarray(sources, dtype=INDEX_DTYPE).ravel()
        dst = np.asarray(targets, dtype=INDEX_DTYPE).ravel()
        if src.shape != dst.shape:
            raise ContractViolation("sources and targets differ in length")
        return cls.from_device(DeviceGraph.from_edges(int(n), src, dst))

    @classmethod
    def from_device(cls, dev: "DeviceGraph"):
        """Wrap a graph that lives on the device (device ingestion, R-MAT)."""
        g = cls.__new__(cls)
        g._dev = dev
        g.n = dev.n
        g._adj = None
        return g

    @property
    def adjacency(self) -> SparseMatrix:
        return self.host_adjacency()

    def host_adjacency(self) -> SparseMatrix:
        if self._adj is None:
            rowptr = self._dev.rowptr.cpu().numpy()
            col = self._dev.col[: self._dev.nnz].cpu().numpy().astype(INDEX_DTYPE)
            self._adj = SparseMatrix(self.n, self.n, rowptr, col, np.ones(col.shape[0]),
                                     validate=False)
        return self._adj

    def device(self) -> "DeviceGraph":
        if self._dev is None:
            A = self._adj
            self._dev = DeviceGraph.upload(self.n, A.row_offsets, A.col_indices)
        return self._dev

    def degrees(self):
        return self.host_adjacency().row_nnz()

    def has_edge(self, u, v):
        cols = self.host_adjacency().row_cols(u)
        i = np.searchsorted(cols, v)
        return bool(i < len(cols) and cols[i] == v)

    def __repr__(self):
        nnz = self._adj.nnz if self._adj is not None else self._dev.nnz
        return f"Graph(n={self.n}, edges={nnz})"


class DeviceGraph:
    """Adjacency in HBM: rowptr int64[n+1], col int32[nnz + GB_COL_PAD]
    (16-B aligned, padded for 16-B streaming loads), plus the C-ABI handle
    owning the per-degree exact-replay tables."""

    def __init__(self, n, rowptr, col, nnz):
        from . import _lib

        self.n = int(n)
        self.nnz = int(nnz)
        self.rowptr = rowptr
        self.col = col
        h = _lib.ctypes.c_void_p()
        _lib.check(_lib.lib().gb_graph_create(self.n, self.nnz, _lib.ptr(rowptr), _lib.ptr(col),
                                              _lib.stream_ptr(), _lib.ctypes.byref(h)),
                   "gb_graph_create")
        self.handle = h
        md, sl = _lib.ctypes.c_int64(), _lib.ctypes.c_int64()
        _lib.check(_lib.load().gb_graph_info(h, _lib.ctypes.byref(md), _lib.ctypes.byref(sl)))
        self.max_degree = int(md.value)
        self.table_slots = int(sl.value)

    @classmethod
    def upload(cls, n, rowptr, col):
        import torch

        from . import _lib

        nnz = int(len(col))
        d_ptr = torch.as_tensor(np.array(rowptr, dtype=np.int64)).cuda()
        d_col = torch.zeros(nnz + _lib.GB_COL_PAD, dtype=torch.int32, device="cuda")
        if nnz:
            d_col[:nnz] = torch.as_tensor(np.asarray(col, dtype=np.int32)).cuda()
        return cls(n, d_ptr, d_col, nnz)

    @classmethod
    def from_edges(cls, n, src, dst):
        """COO (host int64 arrays) -> device CSR by the library's radix sort
        and duplicate collapse (gb_csr_from_edges)."""
        import ctypes

        import torch

        from . import _lib

        if n < 1:
            raise ContractViolation("graph needs at least one vertex")
        L = _lib.lib()
        m = int(src.shape[0])
        d_src = torch.as_tensor(src).cuda()
        d_dst = torch.as_tensor(dst).cuda()
        rowptr = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        col = torch.zeros(m + _lib.GB_COL_PAD, dtype=torch.int32, device="cuda")
        ws = torch.empty(max(int(L.gb_csr_from_edges_workspace(n, m)), 1), dtype=torch.uint8,
                         device="cuda")
        nnz = ctypes.c_int64()
        _lib.check(L.gb_csr_from_edges(n, m, _lib.ptr(d_src), _lib.ptr(d_dst), _lib.ptr(rowptr),
                                       _lib.ptr(col), ctypes.byref(nnz), _lib.ptr(ws),
                                       ws.numel(), _lib.stream_ptr()), "gb_csr_from_edges")
        return cls(n, rowptr, col, int(nnz.value))

    @classmethod
    def from_tensors(cls, n, rowptr, col_padded, nnz):
        return cls(n, rowptr, col_padded, nnz)

    def __del__(self):
        try:
            from . import _lib

            if getattr(self, "handle", None):
                _lib.load().gb_graph_destroy(self.handle)
        except Exception:
            pass


# -- the reference sparse.py kernels, computed on the GPU (ops.py) --------------


def spgemm(left, right):
    from .ops import spgemm as _f

    return _f(left, right)


def add(left, right):
    from .ops import add as _f

    return _f(left, right)


def norm_rows_sage(P):
    from .ops import norm_rows_sage as _f

    return _f(P)


def norm_rows_ladies(P):
    from .ops import norm_rows_ladies as _f

    return _f(P)


def vstack(blocks, n_cols=None):
    from .ops import vstack as _f

    return _f(blocks, n_cols)


def block_diag(blocks):
    from .ops import block_diag as _f

    return _f(blocks)


def compact_columns(M):
    from .ops import compact_columns as _f

    return _f(M)


def expand_row_extraction(Q):
    from .ops import expand_row_extraction as _f

    return _f(Q)


def column_window(M, lo, hi):
    from .ops import column_window as _f

    return _f(M, lo, hi)


def rows_subset(M, rows):
    from .ops import rows_subset as _f

    return _f(M, rows)


def build_column_extraction(sampled_cols, n):
    from .ops import build_column_extraction as _f

    return _f(sampled_cols, n)
