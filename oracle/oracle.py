"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes front end of oracle/liboracle.so (oracle/csrc/oracle.c), the plain-C
restatement of the reference bulk sampler.  Imported only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.

Epoch results are returned as `EpochArrays`: one dict per layer holding the
reference `LayerSample` fields (`pkg/src/gnnbulk/sampler.py:240-261`) as flat
numpy arrays (CSR pointer/column arrays, ragged per-batch vertex lists as
offsets + concatenation).  The same structure is produced from the golden
fixtures (`load_golden`) and from the CUDA path (`paper_2311_02909_b200`
`SampledEpoch.to_arrays()`), and `compare_epochs` checks them field by field
the way reference `SampledEpoch.equals` does (`sampler.py:279-306`).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

LAYER_KEYS = (
    "frontier_shape", "frontier_ptr", "frontier_col",
    "adj_shape", "adj_ptr", "adj_col",
    "rowv_off", "rowv_cat", "colv_off", "colv_cat", "sampv_off", "sampv_cat",
)


class _CSR(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
        ("ptr", ctypes.POINTER(ctypes.c_int64)), ("col", ctypes.POINTER(ctypes.c_int32)),
    ]


class _Layer(ctypes.Structure):
    _fields_ = [
        ("frontier", _CSR), ("adj", _CSR),
        ("rowv_off", ctypes.POINTER(ctypes.c_int64)), ("rowv", ctypes.POINTER(ctypes.c_int32)),
        ("colv_off", ctypes.POINTER(ctypes.c_int64)), ("colv", ctypes.POINTER(ctypes.c_int32)),
        ("sampv_off", ctypes.POINTER(ctypes.c_int64)), ("sampv", ctypes.POINTER(ctypes.c_int32)),
    ]


class _Epoch(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int64), ("k", ctypes.c_int64), ("status", ctypes.c_int64),
        ("layers", ctypes.POINTER(_Layer)),
    ]


def build():
    """Compile liboracle.so with the committed Makefile (gcc, OpenMP)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        i64, u64, p = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        L.orc_sage_bulk.restype = ctypes.POINTER(_Epoch)
        L.orc_sage_bulk.argtypes = [i64, p, p, i64, p, p, i64, i64, p, u64, u64, i64, ctypes.c_int]
        L.orc_ladies_bulk.restype = ctypes.POINTER(_Epoch)
        L.orc_ladies_bulk.argtypes = [i64, p, p, i64, p, p, i64, p, u64, u64, i64, ctypes.c_int]
        L.orc_epoch_free.argtypes = [ctypes.POINTER(_Epoch)]
        L.orc_uniform.restype = ctypes.c_double
        L.orc_uniform.argtypes = [u64, u64, u64, u64, u64]
        L.orc_its_sample_row.restype = i64
        L.orc_its_sample_row.argtypes = [p, i64, i64, p, p]
        L.orc_segment_sum.restype = ctypes.c_double
        L.orc_segment_sum.argtypes = [p, i64]
        L.orc_rmat_graph.restype = i64
        L.orc_rmat_graph.argtypes = [u64, i64, i64, ctypes.c_int, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double,
                                     ctypes.POINTER(ctypes.POINTER(ctypes.c_int64)),
                                     ctypes.POINTER(ctypes.POINTER(ctypes.c_int32))]
        L.orc_free.argtypes = [p]
        _LIB = L
    return _LIB


def rmat_graph(n, m, symmetric=True, seed=0, a=0.57, b=0.19, c=0.19):
    """Host restatement of the library's synthetic graph (gb_rmat_graph,
    oracle/csrc/gen.c): (rowptr int64[n+1], col int32[nnz])."""
    L = lib()
    rp = ctypes.POINTER(ctypes.c_int64)()
    cp = ctypes.POINTER(ctypes.c_int32)()
    nnz = L.orc_rmat_graph(int(seed), int(n), int(m), int(bool(symmetric)), a, b, c,
                           ctypes.byref(rp), ctypes.byref(cp))
    if nnz < 0:
        raise MemoryError("oracle rmat_graph: allocation failed")
    rowptr = np.ctypeslib.as_array(rp, shape=(int(n) + 1,)).copy()
    col = np.ctypeslib.as_array(cp, shape=(max(int(nnz), 1),))[: int(nnz)].copy()
    L.orc_free(ctypes.cast(rp, ctypes.c_void_p))
    L.orc_free(ctypes.cast(cp, ctypes.c_void_p))
    return rowptr, col


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def _unpack(ep_ptr):
    ep = ep_ptr.contents
    if ep.status != 0:
        code = int(ep.status)
        lib().orc_epoch_free(ep_ptr)
        raise ValueError(f"oracle contract violation (code {code})")
    k = int(ep.k)
    layers = []
    for li in range(int(ep.n_layers)):
        L = ep.layers[li]
        d = {}
        for name, c in (("frontier", L.frontier), ("adj", L.adj)):
            d[name + "_shape"] = np.array([c.n_rows, c.n_cols], dtype=np.int64)
            d[name + "_ptr"] = _arr(c.ptr, c.n_rows + 1, np.int64)
            d[name + "_col"] = _arr(c.col, c.nnz, np.int64)
        for name, off, cat in (("rowv", L.rowv_off, L.rowv), ("colv", L.colv_off, L.colv),
                               ("sampv", L.sampv_off, L.sampv)):
            o = _arr(off, k + 1, np.int64)
            d[name + "_off"] = o
            d[name + "_cat"] = _arr(cat, int(o[-1]) if k else 0, np.int64)
        layers.append(d)
    lib().orc_epoch_free(ep_ptr)
    return layers


def _csr_args(rowptr, col):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    return rowptr, col


def _batch_args(batches):
    arrs = [np.asarray(b, dtype=np.int64) for b in batches]
    off = np.zeros(len(arrs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(a) for a in arrs])
    cat = np.concatenate(arrs) if arrs else np.zeros(0, dtype=np.int64)
    return off, np.ascontiguousarray(cat)


def sage_bulk(n, rowptr, col, batches, batch_size, fanouts, seed, epoch=0,
              batch_offset=0, threads=0):
    """Oracle SAGE sample_epoch_bulk (sampler.py:325-387) -> list of layer dicts."""
    rowptr, col = _csr_args(rowptr, col)
    off, cat = _batch_args(batches)
    f = np.ascontiguousarray(fanouts, dtype=np.int64)
    ep = lib().orc_sage_bulk(
        n, rowptr.ctypes.data, col.ctypes.data, len(batches), off.ctypes.data,
        cat.ctypes.data, batch_size, len(f), f.ctypes.data, seed, epoch, batch_offset,
        threads)
    return _unpack(ep)


def ladies_bulk(n, rowptr, col, batches, fanouts, seed, epoch=0, batch_offset=0,
                threads=0):
    """Oracle LADIES sample_epoch_bulk (sampler.py:325-387) -> list of layer dicts."""
    rowptr, col = _csr_args(rowptr, col)
    off, cat = _batch_args(batches)
    f = np.ascontiguousarray(fanouts, dtype=np.int64)
    ep = lib().orc_ladies_bulk(
        n, rowptr.ctypes.data, col.ctypes.data, len(batches), off.ctypes.data,
        cat.ctypes.data, len(f), f.ctypes.data, seed, epoch, batch_offset, threads)
    return _unpack(ep)


def its_sample_row(probs, s, us):
    """Oracle its_sample_row (sampler.py:157-189) fed explicit uniforms."""
    probs = np.ascontiguousarray(probs, dtype=np.float64)
    us = np.ascontiguousarray(us, dtype=np.float64)
    out = np.zeros(max(len(probs), 1), dtype=np.int64)
    t = lib().orc_its_sample_row(probs.ctypes.data, len(probs), s, us.ctypes.data,
                                 out.ctypes.data)
    return out[:t].copy()


def uniform(seed, epoch, depth, row, t):
    return lib().orc_uniform(seed, epoch, depth, row, t)


# -- golden fixtures ----------------------------------------------------------


def load_golden(path, prefix=""):
    """Load an epoch fixture written by tests/golden/make_golden.py (keys
    under `prefix` for the epochs inside pipeline.npz)."""
    z = np.load(path)
    if prefix:
        z = {k[len(prefix):]: v for k, v in z.items() if k.startswith(prefix)} | {
            k: v for k, v in z.items() if k.startswith("A_")}
    layers = []
    for li in range(int(z["n_layers"])):
        p = f"L{li}_"
        d = {}
        for key in LAYER_KEYS:
            d[key] = z[p + key]
        layers.append(d)
    if prefix:
        return {"n": int(z["A_shape"][0]), "rowptr": z["A_ptr"], "col": z["A_col"],
                "kind": str(z["kind"])}, layers
    g = {
        "n": int(z["A_shape"][0]),
        "rowptr": z["A_ptr"],
        "col": z["A_col"],
        "batches": [z["batches_cat"][z["batches_off"][i]:z["batches_off"][i + 1]]
                    for i in range(len(z["batches_off"]) - 1)],
        "layers_cfg": int(z["cfg"][0]),
        "batch_size": int(z["cfg"][1]),
        "seed": int(z["cfg"][2]),
        "epoch": int(z["cfg"][3]),
        "batch_offset": int(z["cfg"][4]),
        "fanouts": [int(x) for x in z["fanouts"]],
        "kind": str(z["kind"]),
        "spgemm_calls": int(z["spgemm_calls"]),
    }
    return g, layers


def compare_epochs(want, got):
    """Field-by-field bitwise comparison (reference SampledEpoch.equals,
    sampler.py:279-306).  Returns a list of mismatch descriptions."""
    errs = []
    if len(want) != len(got):
        return [f"layer count {len(want)} != {len(got)}"]
    for li, (a, b) in enumerate(zip(want, got)):
        for key in LAYER_KEYS:
            x = np.asarray(a[key], dtype=np.int64)
            y = np.asarray(b[key], dtype=np.int64)
            if x.shape != y.shape or not np.array_equal(x, y):
                errs.append(f"layer {li} {key}: shapes {x.shape} vs {y.shape}")
    return errs
