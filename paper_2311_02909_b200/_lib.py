"""ctypes binding of libgnnbulk_b200.so (the C ABI in include/gnnbulk_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every compute entry point raises immediately.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ContractViolation

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgnnbulk_b200.so")

GB_OK = 0
GB_ERR_CONTRACT = -1
GB_ERR_CUDA = -2
GB_ERR_CAPACITY = -3
GB_ERR_UNSUPPORTED = -4
GB_COL_PAD = 4
GB_SAGE_STREAM = 0
GB_SAGE_PFREE = 1
GB_SAGE_DEDUP = 2

_i64, _u64, _i32, _p = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p


class SageLayerOut(ctypes.Structure):
    _fields_ = [
        ("fptr", _p), ("fcol", _p), ("acol", _p), ("colv", _p),
        ("eoff", _p), ("coloff", _p), ("r_cap", _i64), ("f_cap", _i64),
    ]


class LadiesLayerOut(ctypes.Structure):
    _fields_ = [
        ("fptr", _p), ("fcol", _p), ("aptr", _p), ("acol", _p), ("coloff", _p),
        ("q_cap", _i64), ("f_cap", _i64), ("a_cap", _i64),
    ]


GB_LADIES_EXACT = 0
GB_LADIES_RACE = 1
GB_LADIES_RACE_DENSE = 2

# (name, restype, argtypes) — one line per exported symbol of the header
SIGNATURES = {
    "gb_last_error": (ctypes.c_char_p, []),
    "gb_version": (ctypes.c_int, []),
    "gb_uniforms": (ctypes.c_int, [_u64, _u64, _u64, _p, _p, _i64, _p, _p]),
    "gb_graph_create": (ctypes.c_int, [_i64, _i64, _p, _p, _p, ctypes.POINTER(_p)]),
    "gb_graph_destroy": (ctypes.c_int, [_p]),
    "gb_graph_info": (ctypes.c_int, [_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "gb_sage_bulk_workspace": (ctypes.c_int, [_p, _i64, _i64, _i32, _p, ctypes.POINTER(ctypes.c_size_t)]),
    "gb_sage_bulk": (ctypes.c_int, [_p, _i64, _p, _p, _i64, _i64, _i32, _p, _u64, _u64, _i64,
                                    _i32, ctypes.POINTER(SageLayerOut), _p, _p, ctypes.c_size_t, _p]),
    "gb_sage_bulk_peer": (ctypes.c_int, [_p, _i64, _p, _p, _i64, _i64, _i32, _p, _u64, _u64,
                                         _i64, ctypes.POINTER(SageLayerOut), _p, _p,
                                         ctypes.c_size_t, _i32, _p, _p, _p, _p]),
    "gb_ladies_bulk_workspace": (ctypes.c_int, [_p, _i64, _i64, _i32, _p, _i32,
                                                ctypes.POINTER(ctypes.c_size_t)]),
    "gb_ladies_bulk": (ctypes.c_int, [_p, _i64, _p, _p, _i64, _i32, _p, _u64, _u64, _i64, _i32,
                                      ctypes.POINTER(LadiesLayerOut), _p, _p, ctypes.c_size_t,
                                      _p]),
    "gb_ladies_counts_workspace": (ctypes.c_size_t, [_i64, _i64, _i64]),
    "gb_ladies_counts": (ctypes.c_int, [_i64, _p, _p, _p, _i64, _p, _p, _i64, _p, _p, _p, _p,
                                        ctypes.c_size_t, _p]),
    "gb_ladies_layer_rows": (ctypes.c_int, [_p, _i64, _p, _p, _i64, _p, _p, _i64, _u64, _u64,
                                            _i32, _i64, _i32, _p, _p, _p, ctypes.c_size_t, _p]),
    "gb_ladies_merge_counts_workspace": (ctypes.c_size_t, [_i64, _i64]),
    "gb_ladies_merge_counts": (ctypes.c_int, [_i64, _i64, _p, _i64, _i64, _p, _p, _p, _p,
                                              ctypes.c_size_t, _p]),
    "gb_ladies_race_topk_workspace": (ctypes.c_size_t, [_i64, _i64, _i32]),
    "gb_ladies_race_topk": (ctypes.c_int, [_i64, _p, _p, _p, _i64, _i32, _u64, _u64, _u64, _i64,
                                           _p, _p, _p, _p, ctypes.c_size_t, _p]),
    "gb_ladies_extract_rows": (ctypes.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "gb_take_scan": (ctypes.c_int, [_i64, _p, _p, _i32, _p, _p, _p]),
    "gb_sage_layer_sample_workspace": (ctypes.c_size_t, [_i64, _i64]),
    "gb_sage_layer_sample": (ctypes.c_int, [_p, _i64, _p, _i64, _p, _p, _p, _p, _p, _i32, _i64,
                                            _i64, _u64, _u64, _u64, _i32, _p, _p, ctypes.c_size_t,
                                            _p]),
    "gb_sage_sample_keyed": (ctypes.c_int, [_p, _i64, _p, _p, _p, _p, _p, _p, _p, _i32, _u64, _u64,
                                            _u64, _p, _p]),
    "gb_sage_layer_extract_workspace": (ctypes.c_size_t, [_i64, _i64]),
    "gb_sage_layer_extract": (ctypes.c_int, [_i64, _i64, _p, _p, _p, _i64, _p, _p, _p, _p, _p, _p,
                                             ctypes.c_size_t, _p]),
    "gb_gather_rows": (ctypes.c_int, [_i64, _p, _i64, _p, _p, _p, _p, _p]),
    "gb_gather_features": (ctypes.c_int, [_i64, _p, _i64, _p, _i64, _p, _p]),
    "gb_spmm_rows": (ctypes.c_int, [_i64, _p, _p, _p, _p, _i64, _p, _i64, _p, _p]),
    "gb_first_occurrence": (ctypes.c_int, [_i64, _p, _p, _p, _i64, _i64, _p, _p]),
    "gb_segment_copy": (ctypes.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p]),
    "gb_sage_owner_p2p_workspace": (ctypes.c_size_t, [_i64]),
    "gb_sage_owner_p2p": (ctypes.c_int, [_p, _i64, _p, _p, _p, _p, _i64, _i64, _i32, _p, _i64,
                                         _i64, _p, _p, _i32, _i64, _u64, _u64, _u64, _p,
                                         ctypes.c_size_t, _p]),
    "gb_scan_workspace_bytes": (ctypes.c_size_t, [_i64]),
    "gb_spgemm_bound": (ctypes.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p]),
    "gb_spgemm": (ctypes.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _p, _p, _p, _p, _p,
                                 _p, _p, _p, _p, _p]),
    "gb_csr_add": (ctypes.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _p]),
    "gb_norm_rows": (ctypes.c_int, [_i64, _p, _p, _i32, _p, _p, _p]),
    "gb_its_rows": (ctypes.c_int, [_i64, _p, _p, _i32, _p, _p, _u64, _u64, _u64, _p, _p, _p, _p,
                                   _p, _p]),
    "gb_rmat_edges": (ctypes.c_int, [_u64, _i32, _i64, _i64, _i64, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, _p, _p, _p]),
    "gb_hash64": (ctypes.c_int, [_u64, _p, _i64, _p, _p]),
    "gb_spmm_f64": (ctypes.c_int, [_i64, _p, _p, _p, _p, _i64, _p, _p]),
    "gb_csr_from_edges_workspace": (ctypes.c_size_t, [_i64, _i64]),
    "gb_csr_from_edges": (ctypes.c_int, [_i64, _i64, _p, _p, _p, _p, ctypes.POINTER(_i64), _p,
                                         ctypes.c_size_t, _p]),
    "gb_rmat_graph_workspace": (ctypes.c_size_t, [_i64, _i64, _i32, _i64]),
    "gb_rmat_graph": (ctypes.c_int, [_u64, _i64, _i64, _i32, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, _i64, _p, _p, _i64, _p, _p, ctypes.c_size_t,
                                     _p]),
    "gb_rmat_block": (ctypes.c_int, [_u64, _i64, _i64, _i32, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, _i64, _i64, _i64, _p, _p, _i64, _p, _p,
                                     ctypes.c_size_t, _p]),
    "gb_launch_counter": (ctypes.c_int64, [_i32]),
    "gb_profile_begin": (ctypes.c_int, [_i32]),
    "gb_profile_end": (ctypes.c_int, [_p, _i32, _p]),
}

_LIB = None


def load():
    """Load the shared library (no CUDA needed just to load it)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def lib():
    """The library, for a compute call: requires a CUDA device."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2311_02909_b200 needs a CUDA device (B200); no CPU fallback")
    return load()


def check(rc: int, what: str = ""):
    if rc == GB_OK:
        return
    msg = load().gb_last_error().decode(errors="replace")
    if rc == GB_ERR_CONTRACT:
        raise ContractViolation(msg)
    raise RuntimeError(f"{what}: gnnbulk_b200 error {rc}: {msg}")


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)
