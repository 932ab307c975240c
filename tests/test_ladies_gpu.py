"""LADIES on the GPU: bit-exact replay mode against the reference goldens and
the C oracle; the production exponential-race mode against the exact
successive-sampling law (chi-square at 1%, deterministic seeds)."""

import glob
import itertools
import os

import numpy as np
import pytest
from scipy import stats

from conftest import GOLDEN
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _gb():
    import paper_2311_02909_b200 as gb

    return gb


def _graph(n, rowptr, col):
    gb = _gb()
    return gb.Graph(gb.SparseMatrix(n, n, rowptr, col, np.ones(len(col)), validate=False))


LADIES_GOLDEN = sorted(glob.glob(os.path.join(GOLDEN, "epoch_*ladies*.npz")))


@pytest.mark.parametrize("path", LADIES_GOLDEN, ids=os.path.basename)
def test_ladies_exact_matches_reference_golden(path):
    gb = _gb()
    g, want = O.load_golden(path)
    G = _graph(g["n"], g["rowptr"], g["col"])
    cfg = gb.SamplerConfig.ladies(g["layers_cfg"], g["batch_size"], g["fanouts"][0],
                                  bulk_count=len(g["batches"]), seed=g["seed"])
    ep = gb.sample_epoch_bulk(G, cfg, g["batches"], epoch=g["epoch"],
                              batch_offset=g["batch_offset"], mode="exact")
    assert O.compare_epochs(want, ep.to_arrays()) == []


@pytest.mark.parametrize("case", range(3))
def test_ladies_exact_matches_oracle_random(case):
    gb = _gb()
    from test_sage_gpu import _rmat

    rng = np.random.default_rng(200 + case)
    n, rowptr, col = _rmat(11 + case, 20000 * (case + 1), seed=50 + case)
    G = _graph(n, rowptr, col)
    b, s, k = [(16, 8, 3), (64, 32, 5), (128, 100, 2)][case]
    batches = [rng.permutation(n)[:b] for _ in range(k)]
    cfg = gb.SamplerConfig.ladies(3, b, s, bulk_count=k, seed=case)
    ep = gb.sample_epoch_bulk(G, cfg, batches, epoch=case, batch_offset=7 * case, mode="exact")
    want = O.ladies_bulk(n, rowptr, col, batches, [s] * 3, case, case, 7 * case)
    assert O.compare_epochs(want, ep.to_arrays()) == []


def test_ladies_rejects_duplicates():
    gb = _gb()
    G = gb.Graph.from_edges(6, [0, 1, 2], [1, 2, 0])
    cfg = gb.SamplerConfig.ladies(1, 3, 2)
    with pytest.raises(gb.ContractViolation):
        gb.sample_epoch_bulk(G, cfg, [[1, 1, 2]])


def _figure():
    gb = _gb()
    edges = [(0, 1), (1, 4), (2, 5), (3, 5), (4, 5)]
    src = [u for u, v in edges] + [v for u, v in edges]
    dst = [v for u, v in edges] + [u for u, v in edges]
    return gb.Graph.from_edges(6, src, dst)


def test_ladies_race_first_draw_law():
    """s=1: the pick follows the probability row [1/7,0,1/7,1/7,4/7,0]
    (reference test_sampler.py:314-330, test_acceptance.py:46-59)."""
    gb = _gb()
    G = _figure()
    trials = 40000
    cfg = gb.SamplerConfig.ladies(1, 2, 1, bulk_count=trials, seed=77)
    ep = gb.sample_epoch_bulk(G, cfg, [[1, 5]] * trials, mode="race")
    picks = ep.layers[0].to_arrays()["sampv_cat"]
    assert picks.size == trials
    counts = np.bincount(picks, minlength=6)
    expect = np.array([1, 0, 1, 1, 4, 0]) / 7 * trials
    assert counts[[1, 5]].sum() == 0
    sup = expect > 0
    assert stats.chisquare(counts[sup], f_exp=expect[sup]).pvalue > 0.01


def test_ladies_race_pair_law():
    """s=2 without replacement: the sampled pair {a, b} has probability
    w_a w_b / (1 - w_a) + w_b w_a / (1 - w_b) (successive sampling, the law of
    its_sample_row's remove-and-renormalise loop)."""
    gb = _gb()
    G = _figure()
    trials = 40000
    cfg = gb.SamplerConfig.ladies(1, 2, 2, bulk_count=trials, seed=5)
    ep = gb.sample_epoch_bulk(G, cfg, [[1, 5]] * trials, mode="race")
    a = ep.layers[0].to_arrays()
    cat, off = a["sampv_cat"], a["sampv_off"]
    assert np.all(np.diff(off) == 2)
    w = {0: 1 / 7, 2: 1 / 7, 3: 1 / 7, 4: 4 / 7}
    pairs = list(itertools.combinations(sorted(w), 2))
    obs = np.zeros(len(pairs))
    idx = {p: i for i, p in enumerate(pairs)}
    for x, y in cat.reshape(-1, 2):
        obs[idx[(int(x), int(y))]] += 1
    exp = np.array([w[x] * w[y] / (1 - w[x]) + w[y] * w[x] / (1 - w[y]) for x, y in pairs])
    assert abs(exp.sum() - 1) < 1e-12
    assert stats.chisquare(obs, f_exp=exp * trials).pvalue > 0.01


def test_ladies_race_structure_matches_exact_shapes():
    """Race and exact agree on everything that does not depend on the draw:
    row vertices of layer 1, take counts, edges of A_S are real."""
    gb = _gb()
    from test_sage_gpu import _rmat

    rng = np.random.default_rng(9)
    n, rowptr, col = _rmat(12, 40000, seed=9)
    G = _graph(n, rowptr, col)
    batches = [rng.permutation(n)[:64] for _ in range(6)]
    cfg = gb.SamplerConfig.ladies(2, 64, 48, bulk_count=6, seed=1)
    ex = gb.sample_epoch_bulk(G, cfg, batches, mode="exact").to_arrays()
    ra = gb.sample_epoch_bulk(G, cfg, batches, mode="race").to_arrays()
    assert np.array_equal(ex[0]["rowv_cat"], ra[0]["rowv_cat"])
    assert np.array_equal(ex[0]["sampv_off"], ra[0]["sampv_off"])
    A = set(zip(np.repeat(np.arange(n), np.diff(rowptr)).tolist(), col.tolist()))
    for lay in ra:
        rows = lay["rowv_cat"]
        cols = lay["colv_cat"]
        ptr = lay["adj_ptr"]
        shared = lay["adj_shape"][1] != lay["colv_off"][-1] or len(batches) == 1
        for b in range(len(batches)):
            r0, r1 = lay["rowv_off"][b], lay["rowv_off"][b + 1]
            c0 = lay["colv_off"][b]
            for r in range(r0, r1):
                for e in range(ptr[r], ptr[r + 1]):
                    c = lay["adj_col"][e] + (c0 if shared else 0)
                    assert (int(rows[r]), int(cols[c])) in A


@pytest.mark.parametrize("scale,edges,k,b,layers,s", [(16, 300000, 24, 256, 2, 128),
                                                      (12, 30000, 5, 64, 3, 48),
                                                      (5, 60, 3, 4, 2, 3),
                                                      (22, 200000, 4, 64, 2, 32)])
def test_ladies_race_tiled_equals_dense(scale, edges, k, b, layers, s):
    """The production race (column tiles in shared memory: dense and sparse
    tiles — the scale-22 case is sparse) selects exactly what the
    dense-counter race selects: same keys, same (key, v) order."""
    gb = _gb()
    from test_sage_gpu import _rmat

    rng = np.random.default_rng(scale)
    n, rowptr, col = _rmat(scale, edges, seed=scale)
    G = _graph(n, rowptr, col)
    batches = [np.sort(rng.permutation(n)[: rng.integers(1, b + 1)]) for _ in range(k)]
    cfg = gb.SamplerConfig.ladies(layers, b, s, bulk_count=k, seed=3)
    tiled = gb.sample_epoch_bulk(G, cfg, batches, mode="race", epoch=2, batch_offset=7)
    dense = gb.sample_epoch_bulk(G, cfg, batches, mode="race_dense", epoch=2, batch_offset=7)
    assert O.compare_epochs(dense.to_arrays(), tiled.to_arrays()) == []


def _inclusion_table(race, exact, e, min_cell=20):
    """2 x C contingency table of inclusion counts: vertices expected to be
    picked often are their own cells, the rest pooled by count e_v (weight
    class), classes merged upward until every cell holds >= min_cell."""
    tot = race + exact
    own = tot >= 4 * min_cell
    cells_r, cells_x = list(race[own]), list(exact[own])
    rest = ~own & (e > 0)
    classes = np.unique(e[rest])
    acc_r = acc_x = 0
    for c in classes:
        m = rest & (e == c)
        acc_r += int(race[m].sum())
        acc_x += int(exact[m].sum())
        if acc_r >= min_cell and acc_x >= min_cell:
            cells_r.append(acc_r)
            cells_x.append(acc_x)
            acc_r = acc_x = 0
    if acc_r or acc_x:
        cells_r[-1] += acc_r
        cells_x[-1] += acc_x
    return np.array([cells_r, cells_x], dtype=np.float64)


@pytest.mark.parametrize("bias", ["uniform", "degree"])
def test_ladies_race_inclusion_law_at_scale(bias):
    """Production race (column tiles, E/e^2 keys) against the bit-exact
    replay of its_sample_row (sampler.py:157-189, bit-exact with the
    reference goldens above) at a cfg3-like size: one P row with >= 10^5
    candidates, s = 512 draws, hundreds of independent repetitions (the same
    batch repeated across the bulk: keys differ per batch index).  Per-vertex
    inclusion frequencies (hub vertices as their own cells, the rest pooled
    by weight class e_v) must agree by a chi-square contingency test at 1%.
    'degree' draws the batch by degree (hub-biased, like layers >= 2 of a
    LADIES bulk): heavy-tailed counts e_v."""
    gb = _gb()
    from test_sage_gpu import _rmat

    n, rowptr, col = _rmat(18, 1_200_000, seed=18)
    G = _graph(n, rowptr, col)
    rng = np.random.default_rng(31 if bias == "uniform" else 32)
    deg = np.diff(rowptr)
    b, s, k = (32768 if bias == "uniform" else 8192), 512, 128
    p = None if bias == "uniform" else deg / deg.sum()
    batch = np.sort(rng.choice(n, b, replace=False, p=p))
    e = np.bincount(np.concatenate([col[rowptr[u]:rowptr[u + 1]] for u in batch]), minlength=n)
    assert (e > 0).sum() >= 100_000
    cfg = gb.SamplerConfig.ladies(1, b, s, bulk_count=k, seed=11)

    def counts(mode, bulks, epoch0):
        c = np.zeros(n, np.int64)
        for ep in range(epoch0, epoch0 + bulks):
            lay = gb.sample_epoch_bulk(G, cfg, [batch] * k, epoch=ep, mode=mode).to_arrays()[0]
            assert np.all(np.diff(lay["sampv_off"]) == s)
            c += np.bincount(lay["sampv_cat"], minlength=n)
        return c

    race = counts("race", 6, 100)
    exact = counts("exact", 3, 200)
    assert race.sum() == 6 * k * s and exact.sum() == 3 * k * s
    assert np.all(race[e == 0] == 0) and np.all(exact[e == 0] == 0)
    table = _inclusion_table(race, exact, e)
    assert table.shape[1] >= 20
    chi2, pval, dof, _ = stats.chi2_contingency(table)
    assert pval > 0.01, (chi2, dof, pval)


def test_ladies_bulk_sampler_public_api():
    """BulkSampler drives the LADIES path too: host-staged epochs (and the
    streamed ones) equal sample_epoch_bulk, reference-typed fields read as
    zero-copy views."""
    gb = _gb()
    from paper_2311_02909_b200.engine import BulkSampler
    from test_sage_gpu import _rmat

    rng = np.random.default_rng(21)
    n, rowptr, col = _rmat(12, 40000, seed=21)
    G = _graph(n, rowptr, col)
    cfg = gb.SamplerConfig.ladies(3, 64, 32, bulk_count=6, seed=4)
    jobs = [([np.sort(rng.permutation(n)[: rng.integers(1, 65)]) for _ in range(6)], 6 * j)
            for j in range(3)]
    for mode in ("race", "exact"):
        bs = BulkSampler(G, cfg, mode=mode)
        want = [gb.sample_epoch_bulk(G, cfg, b, epoch=1, batch_offset=o, mode=mode)
                for b, o in jobs]
        got = [bs.sample(b, epoch=1, batch_offset=o) for b, o in jobs]
        streamed = list(bs.sample_stream(jobs, epoch=1))
        for w, g, st in zip(want, got, streamed):
            assert O.compare_epochs(w.to_arrays(), g.to_arrays()) == []
            assert O.compare_epochs(w.to_arrays(), st.to_arrays()) == []
            for lw, lg in zip(w.layers, st.layers):
                assert lg.adjacency.equals(lw.adjacency)
                assert lg.frontier.equals(lw.frontier)
                assert all(np.array_equal(a, b) for a, b in zip(lg.col_vertices,
                                                                lw.col_vertices))
