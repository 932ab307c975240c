"""Device graph ingestion (SURVEY.md §8(b) gb_csr_from_edges, §8(f)4):
the radix-sort COO -> CSR against the reference's from_coo(dedup="first")
semantics (host SparseMatrix.from_coo restates sparse.py:82-103), the
device R-MAT generator against its host restatement (oracle/csrc/gen.c,
bit-identical CSR), and load_graph end to end (reference
pkg/tests/test_io.py behaviours)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gb():
    import paper_2311_02909_b200 as gb

    return gb


def _host_csr(n, src, dst):
    gb = _gb()
    A = gb.SparseMatrix.from_coo(n, n, src, dst, np.ones(len(src)), dedup="first")
    return np.asarray(A.row_offsets), np.asarray(A.col_indices)


@pytest.mark.parametrize("n,m,dup", [(1, 0, 0), (5, 0, 0), (2, 3, 1), (1000, 5000, 2000),
                                     (70000, 400000, 100000), (3_000_000, 50, 10),
                                     (1 << 20, 2_000_000, 500_000)])
def test_csr_from_edges_matches_from_coo(n, m, dup):
    gb = _gb()
    rng = np.random.default_rng(n + m)
    src = rng.integers(0, n, m) if n > 1 else np.zeros(m, np.int64)
    dst = rng.integers(0, n, m) if n > 1 else np.zeros(m, np.int64)
    if dup and m:
        pick = rng.integers(0, m, dup)
        src = np.concatenate([src, src[pick]])
        dst = np.concatenate([dst, dst[pick]])
        perm = rng.permutation(src.size)
        src, dst = src[perm], dst[perm]
    G = gb.Graph.from_edges(n, src, dst)
    rp, col = _host_csr(n, src, dst)
    dev = G.device()
    assert dev.nnz == col.size
    assert np.array_equal(dev.rowptr.cpu().numpy(), rp)
    assert np.array_equal(dev.col[: dev.nnz].cpu().numpy(), col)
    assert np.all(dev.col[dev.nnz:].cpu().numpy() == 0)  # streaming-load padding
    assert G.adjacency.equals(gb.SparseMatrix.from_coo(n, n, src, dst, np.ones(src.size),
                                                       dedup="first"))


def test_csr_from_edges_hub_rows_and_order_insensitive():
    gb = _gb()
    rng = np.random.default_rng(5)
    n = 300_000
    hub = np.zeros(200_000, np.int64)  # one row with 200K entries (multi-CTA digit runs)
    src = np.concatenate([hub, rng.integers(0, n, 100_000)])
    dst = np.concatenate([rng.integers(0, n, 200_000), rng.integers(0, n, 100_000)])
    a = gb.Graph.from_edges(n, src, dst)
    perm = rng.permutation(src.size)
    b = gb.Graph.from_edges(n, src[perm], dst[perm])
    assert a.adjacency.equals(b.adjacency)
    rp, col = _host_csr(n, src, dst)
    assert np.array_equal(np.asarray(a.adjacency.col_indices), col)


def test_csr_from_edges_range_errors():
    gb = _gb()
    with pytest.raises(gb.ContractViolation, match="row index"):
        gb.Graph.from_edges(4, [0, 4], [1, 1])
    with pytest.raises(gb.ContractViolation, match="column index"):
        gb.Graph.from_edges(4, [0, 1], [1, -1])
    with pytest.raises(gb.ContractViolation):
        gb.Graph.from_edges(4, [0, 1], [1])


@pytest.mark.parametrize("n,m,sym,seed", [(4096, 30000, True, 3), (4096, 20000, False, 3),
                                          (65536, 1 << 20, True, 0), (100_003, 300_000, True, 9),
                                          (1000, 200, False, 1)])
def test_device_rmat_equals_host_restatement(n, m, sym, seed):
    from oracle import oracle as O
    from paper_2311_02909_b200.graphgen import rmat_device_graph

    dg = rmat_device_graph(n, m, symmetric=sym, seed=seed)
    rp, col = O.rmat_graph(n, m, symmetric=sym, seed=seed)
    assert dg.nnz == (2 * m if sym else m) == rp[-1]
    assert np.array_equal(dg.rowptr.cpu().numpy(), rp)
    assert np.array_equal(dg.col[: dg.nnz].cpu().numpy(), col)


FIGURE = [(0, 1), (1, 0), (1, 4), (4, 1), (2, 5), (5, 2), (3, 5), (5, 3), (4, 5), (5, 4)]


def _write(path, lines):
    path.write_text("\n".join(lines) + "\n")


def test_load_graph_edge_list(tmp_path):
    """reference pkg/tests/test_io.py:TestEdgeList."""
    gb = _gb()
    p = tmp_path / "g.txt"
    _write(p, [f"{u} {v}" for u, v in FIGURE])
    G = gb.load_graph(p)
    assert G.n == 6 and G.degrees().tolist() == [1, 2, 1, 1, 2, 3]
    d = G.adjacency.to_dense()
    assert (d[1] + d[5]).tolist() == [1.0, 0.0, 1.0, 1.0, 2.0, 0.0]
    q = tmp_path / "r.txt"
    _write(q, [f"{u} {v}" for u, v in reversed(FIGURE)] + ["1 4"])
    assert gb.load_graph(q).adjacency.equals(G.adjacency)  # order, duplicates
    _write(p, ["# n=4"])
    E = gb.load_graph(p)
    assert E.n == 4 and E.adjacency.nnz == 0
    _write(p, ["0 1", "2 1"])
    S = gb.load_graph(p, direction="symmetrize")
    assert S.has_edge(1, 0) and S.has_edge(1, 2) and S.adjacency.nnz == 4


def test_save_load_matrix_market_round_trip(tmp_path):
    gb = _gb()
    from paper_2311_02909_b200.graphgen import rmat_device_graph

    G = gb.Graph.from_device(rmat_device_graph(300, 900, symmetric=True, seed=2))
    p = tmp_path / "g.mtx"
    gb.save_graph(G, p)
    H = gb.load_graph(p, fmt="matrix-market")
    assert H.n == G.n and H.adjacency.equals(G.adjacency)
