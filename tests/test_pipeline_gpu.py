"""Epoch pipeline on the GPU (reference pipeline.py): aggregation products,
the bulk propagation chain, feature fetch and run_epoch accounting, against
the numpy/scipy restatement in oracle/pipeline_ref.py (float64; the device
computes in float32, tolerance 1e-5 relative)."""

import numpy as np
import pytest

from oracle import pipeline_ref as PR

pytestmark = pytest.mark.gpu

RTOL = 1e-5


def _gb():
    import paper_2311_02909_b200 as gb

    return gb


def _graph(scale, edges, seed):
    from test_sage_gpu import _graph as g, _rmat

    n, rowptr, col = _rmat(scale, edges, seed=seed)
    return n, g(n, rowptr, col)


def _close(got, want):
    scale = np.maximum(np.abs(want), 1.0)
    assert np.all(np.abs(got - want) <= RTOL * scale), float(np.max(np.abs(got - want) / scale))


@pytest.mark.parametrize("f", [1, 3, 64, 130])
def test_forward_aggregate_matches_scipy(f):
    gb = _gb()
    rng = np.random.default_rng(f)
    R, C = 300, 200
    dense = rng.random((R, C)) < 0.05
    dense[7] = False  # an empty row
    A = gb.SparseMatrix.from_dense(dense.astype(np.float64)) if hasattr(gb.SparseMatrix, "from_dense") \
        else None
    if A is None:
        rows, cols = np.nonzero(dense)
        ptr = np.zeros(R + 1, np.int64)
        np.cumsum(np.bincount(rows, minlength=R), out=ptr[1:])
        A = gb.SparseMatrix(R, C, ptr, cols, np.ones(cols.size))
    H = rng.random((C, f)).astype(np.float32).astype(np.float64)
    got = gb.forward_aggregate(A, H)
    want = PR.forward_aggregate(R, C, A.row_offsets, A.col_indices, H)
    assert got.shape == (R, f) and got.dtype == np.float64
    _close(got, want)
    # any values, float64, the reference's scipy order: bit-identical
    W = gb.SparseMatrix(R, C, A.row_offsets, A.col_indices, rng.standard_normal(A.nnz))
    Hn = rng.standard_normal((C, f))
    assert np.array_equal(gb.forward_aggregate(W, Hn), W.to_scipy() @ Hn)
    with pytest.raises(gb.ContractViolation):
        gb.forward_aggregate(A, H[:-1])


@pytest.mark.parametrize("sampler", ["sage", "ladies"])
def test_propagate_bulk_matches_per_batch_reference(sampler):
    gb = _gb()
    rng = np.random.default_rng(3)
    n, G = _graph(12, 30000, seed=3)
    k = 5
    if sampler == "sage":
        cfg = gb.SamplerConfig.sage(3, 32, (6, 4, 3), bulk_count=k, seed=2)
        batches = [rng.permutation(n)[: rng.integers(1, 33)] for _ in range(k)]
    else:
        cfg = gb.SamplerConfig.ladies(2, 32, 24, bulk_count=k, seed=2)
        batches = [np.sort(rng.permutation(n)[: rng.integers(1, 33)]) for _ in range(k)]
    ep = gb.sample_epoch_bulk(G, cfg, batches, mode="race" if sampler == "ladies" else "dedup")
    layers = ep.to_arrays()
    f = 16
    H = rng.random((n, f)).astype(np.float32).astype(np.float64)
    import torch

    deep = layers[-1]
    X = torch.as_tensor(H[deep["colv_cat"]].astype(np.float32)).cuda()
    Y = gb.propagate_bulk(ep, X).cpu().numpy().astype(np.float64)
    roff = layers[0]["rowv_off"]
    assert Y.shape[0] == roff[-1]
    for b in range(k):
        Xb = H[deep["colv_cat"][deep["colv_off"][b]:deep["colv_off"][b + 1]]]
        want = PR.propagate_batch(layers, b, Xb)
        _close(Y[roff[b]:roff[b + 1]], want)


@pytest.mark.parametrize("p,c", [(1, 1), (2, 1), (4, 2)])
def test_fetch_features_rows_and_ledger(p, c):
    gb = _gb()
    from paper_2311_02909_b200.dist import CommLedger, ProcessGrid

    rng = np.random.default_rng(p)
    n, f = 1000, 7
    H = rng.random((n, f))
    grid = ProcessGrid(p, c)
    Hp = gb.FeaturePartition.partition(H, grid)
    verts = rng.integers(0, n, size=300)
    for requester in range(p):
        led = CommLedger(p)
        got = gb.fetch_features(verts, Hp, grid, led, requester)
        assert got.dtype == np.float64
        assert np.array_equal(got, H[verts])  # float64 rows, bit for bit
        want = PR.fetch_words(verts, Hp.row_starts, f, grid.rows, c, requester)
        for r in range(p):
            m, w = want.get(r, (0, 0))
            assert led.messages("all-to-allv", r) == m
            assert led.words("all-to-allv", r) == w
    with pytest.raises(gb.ContractViolation):
        gb.fetch_features([n], Hp, grid)


def test_run_epoch_accounting():
    gb = _gb()
    from paper_2311_02909_b200.dist import ProcessGrid

    n, G = _graph(11, 12000, seed=4)
    cfg = gb.SamplerConfig.sage(2, 64, (5, 3), bulk_count=8, seed=6)
    H = np.random.default_rng(0).random((n, 8))
    for p, c, mode in [(1, 1, "replicated"), (4, 1, "replicated"), (4, 2, "partitioned")]:
        grid = ProcessGrid(p, c)
        rep = gb.run_epoch(G, gb.FeaturePartition.partition(H, grid), cfg, grid, mode=mode,
                           epoch=1)
        nb = -(-n // 64)
        assert rep.n_batches == nb and rep.chunks == -(-nb // 8)
        assert rep.spgemm_calls == 2 * rep.chunks
        want = [0] * p
        for start in range(0, nb, 8):
            size = min(8, nb - start)
            for local in range(size):
                want[PR.trainer_of_batch(local, size, p, grid.rows, c, mode == "replicated")] += 1
        assert rep.batches_per_process == want
        assert set(rep.durations) == {"sample", "fetch", "propagate"}


def _pipeline_golden():
    import os

    from conftest import GOLDEN

    return os.path.join(GOLDEN, "pipeline.npz"), dict(np.load(os.path.join(GOLDEN,
                                                                         "pipeline.npz")))


@pytest.mark.parametrize("kind", ["sage", "ladies"])
def test_propagate_matches_reference_outputs(kind):
    """The device pipeline against the reference's own fetch_features +
    _propagate_batch outputs (tests/golden/pipeline.npz, make_golden.py):
    the bulk's epoch is bit-exact with the reference epoch, the propagated
    rows agree within 1e-5 (device fp32, reference fp64)."""
    import torch

    from oracle import oracle as O

    gb = _gb()
    path, z = _pipeline_golden()
    g, want_layers = O.load_golden(path, prefix=f"{kind}_ep_")
    G = gb.Graph(gb.SparseMatrix(g["n"], g["n"], g["rowptr"], g["col"], np.ones(len(g["col"])),
                                 validate=False))
    c = z[f"{kind}_cfg"]
    off, cat = z[f"{kind}_batches_off"], z[f"{kind}_batches_cat"]
    batches = [cat[off[i]:off[i + 1]] for i in range(len(off) - 1)]
    if kind == "sage":
        cfg = gb.SamplerConfig.sage(int(c[0]), int(c[1]), tuple(int(x) for x in c[3:]),
                                    bulk_count=len(batches), seed=int(c[2]))
        mode = "dedup"
    else:
        cfg = gb.SamplerConfig.ladies(int(c[0]), int(c[1]), int(c[3]), bulk_count=len(batches),
                                      seed=int(c[2]))
        mode = "exact"
    ep = gb.sample_epoch_bulk(G, cfg, batches, epoch=2, batch_offset=3, mode=mode)
    assert O.compare_epochs(want_layers, ep.to_arrays()) == []
    H = z["H"]
    deep = want_layers[-1]
    X = torch.as_tensor(H[deep["colv_cat"]].astype(np.float32)).cuda()
    Y = gb.propagate_bulk(ep, X).cpu().numpy().astype(np.float64)
    Yw, Yoff = z[f"{kind}_Y"], z[f"{kind}_Yoff"]
    roff = want_layers[0]["rowv_off"]
    for b in range(len(batches)):
        _close(Y[roff[b]:roff[b + 1]], Yw[Yoff[b]:Yoff[b + 1]])


def test_fetch_and_run_epoch_match_reference_ledger():
    """fetch_features on a 4 x 2 grid (rows and all-to-allv ledger) and
    run_epoch's accounting (batches, chunks, spgemm calls, per-process
    counts, ledger messages / words per phase) against the reference's own
    outputs (tests/golden/pipeline.npz)."""
    gb = _gb()
    from paper_2311_02909_b200.dist import PHASES, CommLedger, ProcessGrid

    path, z = _pipeline_golden()
    n = int(z["A_shape"][0])
    G = gb.Graph(gb.SparseMatrix(n, n, z["A_ptr"], z["A_col"], np.ones(len(z["A_col"])),
                                 validate=False))
    H = z["H"]
    grid = ProcessGrid(4, 2)
    Hp = gb.FeaturePartition.partition(H, grid)
    for req in range(4):
        led = CommLedger(4)
        rows = gb.fetch_features(z["fetch_verts"], Hp, grid, led, req)
        assert np.array_equal(rows, H[z["fetch_verts"]])
        for proc in range(4):
            assert led.words(phase="all-to-allv", process=proc) == z["fetch_words"][req, proc]
            assert led.messages(phase="all-to-allv", process=proc) == z["fetch_msgs"][req, proc]
    cfg = gb.SamplerConfig.sage(2, 64, (5, 3), bulk_count=4, seed=6)
    for row in z["run_epoch"]:
        p, c = int(row[0]), int(row[1])
        mode = "replicated" if (p, c) != (4, 2) else "partitioned"
        grid = ProcessGrid(p, c)
        rep = gb.run_epoch(G, gb.FeaturePartition.partition(H, grid), cfg, grid, mode=mode,
                           epoch=1)
        got = [p, c, rep.n_batches, rep.chunks, rep.spgemm_calls]
        got += list(rep.batches_per_process) + [0] * (4 - p)
        got += [rep.ledger.messages(phase=ph) for ph in PHASES]
        got += [rep.ledger.words(phase=ph) for ph in PHASES]
        assert got == [int(x) for x in row], (p, c, mode)
