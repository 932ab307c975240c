"""Distributed API on the device, mirroring the reference acceptance tests
4-7 (pkg/tests/test_acceptance.py:110-240): serial == distributed for every
grid and mode, staged multiply == dense oracle, sparsity-aware transfers,
traffic within the cost-model band."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _gb():
    import paper_2311_02909_b200 as gb

    return gb


def d_regular(n, d, seed):
    gb = _gb()
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    rows = np.repeat(np.arange(n), d)
    cols = (rows + np.tile(np.arange(1, d + 1), n)) % n
    return gb.Graph.from_edges(n, perm[rows], perm[cols])


@pytest.mark.parametrize("kind", ["sage", "ladies"])
def test_serial_equals_distributed(kind):
    gb = _gb()
    from paper_2311_02909_b200.dist import CommLedger, ProcessGrid, sample_epoch_distributed

    n = 2000
    G = d_regular(n, 6, seed=3)
    rng = np.random.default_rng(3)
    k, b = 8, 4
    batches = [rng.permutation(n)[:b] for _ in range(k)]
    cfg = (gb.SamplerConfig.sage(2, b, (3, 2), bulk_count=k, seed=13) if kind == "sage"
           else gb.SamplerConfig.ladies(2, b, 3, bulk_count=k, seed=13))
    ref = gb.sample_epoch_bulk(G, cfg, batches, mode="exact" if kind == "ladies" else "auto")
    for p, c in ((2, 1), (4, 1), (4, 2), (8, 2)):
        for mode in ("replicated", "partitioned"):
            ep = sample_epoch_distributed(G, cfg, batches, ProcessGrid(p, c), mode=mode,
                                          ledger=CommLedger(p))
            assert ref.equals(ep), (kind, p, c, mode)


def test_staged_spgemm_equals_dense_oracle():
    gb = _gb()
    from paper_2311_02909_b200.dist import (CommLedger, ProcessGrid, partition_block_rows,
                                            replicated_spgemm, spgemm_15d_sparsity_aware)

    rng = np.random.default_rng(5)
    for trial, (p, c) in enumerate([(2, 1), (4, 1), (4, 2), (8, 2)] * 3):
        m, kk, nn = (int(x) for x in rng.integers(8, 40, size=3))
        A = np.where(rng.random((m, kk)) < 0.2, rng.integers(1, 65, (m, kk)) / 64.0, 0.0)
        B = np.where(rng.random((kk, nn)) < 0.2, rng.integers(1, 65, (kk, nn)) / 64.0, 0.0)
        a, bm = gb.SparseMatrix.from_dense(A), gb.SparseMatrix.from_dense(B)
        grid = ProcessGrid(p, c)
        ap = partition_block_rows(a, grid)
        assert np.array_equal(replicated_spgemm(ap, bm, grid).to_matrix().to_dense(), A @ B)
        st = spgemm_15d_sparsity_aware(ap, partition_block_rows(bm, grid), grid, CommLedger(p))
        assert np.array_equal(st.to_matrix().to_dense(), A @ B)


def test_sparsity_aware_transfers_are_exact():
    gb = _gb()
    from paper_2311_02909_b200.dist import (CommLedger, ProcessGrid, partition_block_rows,
                                            spgemm_15d_sparsity_aware)

    rng = np.random.default_rng(6)
    for p, c in ((4, 1), (8, 2), (4, 2)):
        grid = ProcessGrid(p, c)
        q = gb.SparseMatrix.from_dense(np.where(rng.random((4 * grid.rows, 96)) < 0.08, 1.0, 0))
        a = gb.SparseMatrix.from_dense(np.where(rng.random((96, 96)) < 0.1, 1.0, 0.0))
        qp, apart = partition_block_rows(q, grid), partition_block_rows(a, grid)
        trace = []
        spgemm_15d_sparsity_aware(qp, apart, grid, CommLedger(p), trace)
        assert len(trace) == grid.stages * grid.p
        for rec in trace:
            i, _ = grid.coords(rec.consumer)
            lo, hi = apart.block_range(rec.block)
            cols = qp.block(i).col_indices
            assert np.array_equal(rec.requested_cols, np.unique(cols[(cols >= lo) & (cols < hi)]))
            assert rec.words == int(apart.block(rec.block).row_nnz()[rec.requested_cols - lo].sum())


def test_cost_model_band():
    gb = _gb()
    from paper_2311_02909_b200.dist import (CommLedger, ProcessGrid, partition_block_rows,
                                            spgemm_15d_sparsity_aware)

    n, k, b, d = 2**14, 4, 128, 8  # the reference's sizes (test_acceptance.py:204-206)
    G = d_regular(n, d, seed=d)
    rng = np.random.default_rng(d)
    q = gb.sage_seed_matrix(list(rng.permutation(n)[: k * b].reshape(k, b)), n)
    kbd = k * b * d
    for p, c in ((8, 1), (8, 2), (4, 2)):
        grid = ProcessGrid(p, c)
        led = CommLedger(p)
        spgemm_15d_sparsity_aware(partition_block_rows(q, grid),
                                  partition_block_rows(G.adjacency, grid), grid, led)
        for j in range(c):
            words = sum(led.words("row-data", r) for r in grid.col_group(j))
            assert 0.5 * kbd / c <= words <= 2.0 * kbd / c
        if c >= 2:
            for r in range(p):
                assert 0.5 * c * kbd / p <= led.words("all-reduce", r) <= 2.0 * c * kbd / p
