"""CPU checks of the boundary: the C-ABI library loads without a GPU and
exports every symbol include/gnnbulk_b200.h declares, and the ctypes table
covers them all (no compute calls here)."""

import ctypes
import os
import re

from conftest import REPO

HEADER = os.path.join(REPO, "include", "gnnbulk_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "gb_sage_bulk" in syms and "gb_ladies_bulk" in syms and "gb_uniforms" in syms
    assert len(syms) >= 14


def test_library_exports_every_declared_symbol():
    from paper_2311_02909_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert missing == []


def test_ctypes_table_covers_header():
    from paper_2311_02909_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared_symbols()
    _lib.load()  # binds every signature


def test_version_and_error_without_gpu():
    from paper_2311_02909_b200 import _lib

    L = _lib.load()
    assert L.gb_version() >= 1
    assert isinstance(L.gb_last_error(), bytes)


def test_compute_entry_points_fail_loudly_without_cuda():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2311_02909_b200 as gb

    with pytest.raises(RuntimeError):
        gb.Graph.from_edges(4, [0, 1], [1, 0])  # device ingestion, no host fallback
    G = gb.Graph(gb.SparseMatrix(4, 4, [0, 1, 2, 2, 2], [1, 0], [1.0, 1.0]))
    cfg = gb.SamplerConfig.sage(1, 2, 2)
    with pytest.raises(RuntimeError):
        gb.sample_epoch_bulk(G, cfg, [[0, 1]])
