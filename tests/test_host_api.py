"""Host-side API semantics mirrored from the reference tests
(pkg/tests/test_sparse.py, test_sampler.py): containers, config, seed
matrices, keys, batching.  Pure CPU."""

import numpy as np
import pytest

import paper_2311_02909_b200 as gb
from paper_2311_02909_b200.pipeline import make_batches


def test_sparse_invariants():
    with pytest.raises(gb.ContractViolation):
        gb.SparseMatrix(2, 2, [0, 1], [0], [1.0])
    with pytest.raises(gb.ContractViolation):
        gb.SparseMatrix(1, 3, [0, 2], [2, 1], [1.0, 1.0])
    with pytest.raises(gb.ContractViolation):
        gb.SparseMatrix(1, 3, [0, 2], [1, 1], [1.0, 1.0])
    with pytest.raises(gb.ContractViolation):
        gb.SparseMatrix(1, 3, [0, 1], [3], [1.0])
    with pytest.raises(gb.ContractViolation):
        gb.SparseMatrix(1, 3, [0, 1], [0], [np.inf])
    ok = gb.SparseMatrix(2, 3, [0, 2, 3], [1, 2, 0], [1.0, 2.0, 3.0])
    assert ok.nnz == 3 and ok.shape == (2, 3)
    with pytest.raises(ValueError):
        ok.col_indices[0] = 5  # frozen


def test_from_coo_modes():
    s = gb.SparseMatrix.from_coo(2, 2, [0, 0, 1], [1, 1, 0], [1.0, 2.0, 3.0])
    assert s.to_dense().tolist() == [[0.0, 3.0], [3.0, 0.0]]
    f = gb.SparseMatrix.from_coo(2, 2, [0, 0, 1], [1, 1, 0], [1.0, 2.0, 3.0], dedup="first")
    assert f.nnz == 2


def test_graph_figure_degrees():
    edges = [(0, 1), (1, 4), (2, 5), (3, 5), (4, 5)]
    src = [u for u, v in edges] + [v for u, v in edges]
    dst = [v for u, v in edges] + [u for u, v in edges]
    # host container path (from_edges builds on the device: tests/test_ingest_gpu.py)
    G = gb.Graph(gb.SparseMatrix.from_coo(6, 6, src, dst, np.ones(len(src)), dedup="first"))
    assert G.degrees().tolist() == [1, 2, 1, 1, 2, 3]  # reference test_io.py:36-44
    assert G.has_edge(5, 4) and not G.has_edge(0, 5)
    with pytest.raises(gb.ContractViolation):
        gb.Graph(gb.SparseMatrix(1, 2, [0, 1], [1], [1.0]))
    with pytest.raises(gb.ContractViolation):
        gb.Graph(gb.SparseMatrix(2, 2, [0, 1, 1], [1], [2.0]))


def test_sampler_config():
    cfg = gb.SamplerConfig.sage(3, 4, (15, 10, 5))
    assert [cfg.rows_per_batch(d) for d in (1, 2, 3)] == [4, 60, 600]
    assert gb.SamplerConfig.ladies(3, 4, 5).rows_per_batch(3) == 1
    for bad in (lambda: gb.SamplerConfig.sage(0, 2, ()),
                lambda: gb.SamplerConfig.sage(1, 0, 2),
                lambda: gb.SamplerConfig.ladies(1, 2, 0),
                lambda: gb.SamplerConfig.sage(2, 2, (3,))):
        with pytest.raises(gb.ContractViolation):
            bad()


def test_seed_matrices():
    q = gb.sage_seed_matrix([[1, 5], [0, 2]], 6)
    assert q.shape == (4, 6) and q.row_cols(2).tolist() == [0]
    l = gb.ladies_seed_matrix([[5, 1]], 6)
    assert l.row_cols(0).tolist() == [1, 5]
    assert gb.ladies_seed_matrix([[3], [1]], 6).equals(gb.sage_seed_matrix([[3], [1]], 6))
    with pytest.raises(gb.ContractViolation):
        gb.sage_seed_matrix([[6]], 6)
    with pytest.raises(gb.ContractViolation):
        gb.ladies_seed_matrix([[1, 1]], 6)


def test_global_row_keys():
    cfg = gb.SamplerConfig.sage(2, 3, (2, 2))
    keys = gb.global_row_keys(cfg, 2, [4, 5], [6, 1])
    assert keys.tolist() == [24, 25, 26, 27, 28, 29, 30]
    with pytest.raises(gb.ContractViolation):
        gb.global_row_keys(cfg, 1, [0], [4])


def test_make_batches_matches_reference_recipe():
    b = make_batches(np.arange(10), 4, seed=1, epoch=2)
    order = np.random.Generator(np.random.PCG64(
        np.random.SeedSequence([1, 0x6261746368, 2]))).permutation(10)
    assert [x.tolist() for x in b] == [order[0:4].tolist(), order[4:8].tolist(),
                                       order[8:].tolist()]


def test_epoch_plan_and_trainers_match_reference_rules():
    from oracle import pipeline_ref as PR
    from paper_2311_02909_b200.dist import ProcessGrid
    from paper_2311_02909_b200.pipeline import EpochPlan, _trainer_of_batch

    plan = EpochPlan.build(10, 4)
    assert plan.chunks == ((0, 4), (4, 8), (8, 10)) and plan.rounds == 3
    assert EpochPlan.build(0, 3).chunks == ()
    import pytest
    from paper_2311_02909_b200 import ContractViolation

    with pytest.raises(ContractViolation):
        EpochPlan.build(5, 0)
    for p, c in [(1, 1), (4, 1), (4, 2), (8, 2)]:
        grid = ProcessGrid(p, c)
        for size in (1, 3, 8, 13):
            for local in range(size):
                for mode, rep in (("replicated", True), ("partitioned", False)):
                    assert _trainer_of_batch(local, size, grid, mode) == \
                        PR.trainer_of_batch(local, size, p, grid.rows, c, rep)
