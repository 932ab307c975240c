"""Parity of the CUDA SAGE bulk sampler (both kernel modes) with the oracle.

Bit-exact: the reference's own outputs (golden fixtures, reference run with
the injected uniforms) and the C oracle on seeded random graphs."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O
from oracle.philox import uniforms as np_uniforms

pytestmark = pytest.mark.gpu

MODES = ("stream", "pfree", "dedup")


def _pkg():
    import paper_2311_02909_b200 as gb

    return gb


def _graph(n, rowptr, col):
    gb = _pkg()
    A = gb.SparseMatrix(n, n, rowptr, col, np.ones(len(col)), validate=False)
    return gb.Graph(A)


def test_device_uniforms_match_oracle():
    from paper_2311_02909_b200 import ops

    rows = np.array([0, 1, 5, 2**33 + 7, 16_700_000_000] * 8)
    t = np.repeat(np.arange(8), 5)
    got = ops.uniforms(3, 1, 2, rows, t)
    assert np.array_equal(got, np_uniforms(3, 1, 2, rows, t))


SAGE_GOLDEN = [p for p in sorted(glob.glob(os.path.join(GOLDEN, "epoch_*sage*.npz")))]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("path", SAGE_GOLDEN, ids=os.path.basename)
def test_sage_matches_reference_golden(path, mode):
    gb = _pkg()
    g, want = O.load_golden(path)
    G = _graph(g["n"], g["rowptr"], g["col"])
    cfg = gb.SamplerConfig.sage(g["layers_cfg"], g["batch_size"], tuple(g["fanouts"]),
                                bulk_count=len(g["batches"]), seed=g["seed"])
    ep = gb.sample_epoch_bulk(G, cfg, g["batches"], epoch=g["epoch"],
                              batch_offset=g["batch_offset"], mode=mode)
    assert O.compare_epochs(want, ep.to_arrays()) == []
    assert ep.spgemm_calls == g["spgemm_calls"]


def _rmat(scale, m, seed):
    rng = np.random.default_rng(seed)
    n = 1 << scale
    u = np.zeros(4 * m, np.int64)
    v = np.zeros(4 * m, np.int64)
    for lvl in range(scale):
        r = rng.random(4 * m)
        u |= (r >= 0.76).astype(np.int64) << lvl
        v |= (((r >= 0.57) & (r < 0.76)) | (r >= 0.95)).astype(np.int64) << lvl
    keep = u != v
    src = np.concatenate([u[keep], v[keep]])
    dst = np.concatenate([v[keep], u[keep]])
    key = np.unique(src * n + dst)
    rowptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(key // n, minlength=n), out=rowptr[1:])
    return n, rowptr, (key % n).astype(np.int64)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("case", range(4))
def test_sage_matches_oracle_random(case, mode):
    gb = _pkg()
    rng = np.random.default_rng(100 + case)
    n, rowptr, col = _rmat(12 + case % 2, 30000 * (1 + case), seed=case)
    G = _graph(n, rowptr, col)
    b = [17, 64, 100, 256][case]
    k = [1, 3, 8, 5][case]
    fan = [(15, 10, 5), (3, 2), (25, 1, 32), (10, 10)][case]
    batches = [rng.permutation(n)[: rng.integers(1, b + 1)] for _ in range(k)]
    cfg = gb.SamplerConfig.sage(len(fan), b, fan, bulk_count=k, seed=case * 7 + 1)
    ep = gb.sample_epoch_bulk(G, cfg, batches, epoch=case, batch_offset=3 * case, mode=mode)
    want = O.sage_bulk(n, rowptr, col, batches, b, fan, case * 7 + 1, case, 3 * case)
    assert O.compare_epochs(want, ep.to_arrays()) == []


@pytest.mark.parametrize("mode", MODES)
def test_sage_edge_cases(mode):
    gb = _pkg()
    # isolated vertices, degree == fanout, degree < fanout, duplicates in a
    # batch, an empty batch
    n = 40
    src = [0, 0, 0, 1, 1, 2, 3, 3, 3, 3, 3]
    dst = [1, 2, 3, 0, 4, 0, 5, 6, 7, 8, 9]
    G = gb.Graph.from_edges(n, src, dst)
    A = G.adjacency
    batches = [[0, 1, 2, 3, 39], [], [3, 3, 39, 0]]
    for fan in ((3, 2), (1, 1), (5, 32)):
        cfg = gb.SamplerConfig.sage(2, 5, fan, bulk_count=3, seed=9)
        ep = gb.sample_epoch_bulk(G, cfg, batches, mode=mode)
        want = O.sage_bulk(n, A.row_offsets, A.col_indices, batches, 5, fan, 9)
        assert O.compare_epochs(want, ep.to_arrays()) == []


def test_sage_host_fields_match_reference_types():
    gb = _pkg()
    g, want = O.load_golden(os.path.join(GOLDEN, "epoch_fig_sage.npz"))
    G = _graph(g["n"], g["rowptr"], g["col"])
    cfg = gb.SamplerConfig.sage(2, 2, (2, 2), seed=3)
    ep = gb.sample_epoch_bulk(G, cfg, [[1, 5]])
    layer = ep.layers[0]
    assert layer.frontier.shape == (2, 6)
    assert layer.adjacency.n_rows == 2
    assert np.array_equal(ep.deepest_frontier(0), ep.layers[-1].sampled_vertices[0])
    assert all(isinstance(v, np.ndarray) for v in layer.col_vertices)
    same = gb.sample_epoch_bulk(G, cfg, [[1, 5]], mode="pfree")
    assert ep.equals(same)


def test_sage_rejects_bad_batches():
    gb = _pkg()
    G = gb.Graph.from_edges(6, [0, 1], [1, 0])
    cfg = gb.SamplerConfig.sage(1, 2, 2)
    with pytest.raises(gb.ContractViolation):
        gb.sample_epoch_bulk(G, cfg, [[6]])
    with pytest.raises(gb.ContractViolation):
        gb.sample_epoch_bulk(G, cfg, [[0, 1, 2]])  # longer than batch_size


def test_bulk_sampler_public_api_matches():
    gb = _pkg()
    from paper_2311_02909_b200.engine import BulkSampler

    g, want = O.load_golden(os.path.join(GOLDEN, "epoch_rmat12_sage.npz"))
    G = _graph(g["n"], g["rowptr"], g["col"])
    cfg = gb.SamplerConfig.sage(3, g["batch_size"], tuple(g["fanouts"]),
                                bulk_count=len(g["batches"]), seed=g["seed"])
    for mode in MODES:
        bs = BulkSampler(G, cfg, mode=mode)
        for _ in range(2):
            ep = bs.sample(g["batches"], epoch=g["epoch"])
            assert O.compare_epochs(want, ep.to_arrays()) == []
        dev = bs.sample(g["batches"], epoch=g["epoch"], to_host=False)
        assert O.compare_epochs(want, dev.to_arrays()) == []


def test_bulk_sampler_stream_matches_single_calls():
    """sample_stream (copy of bulk j overlapping bulk j+1) returns exactly
    what one sample() call per bulk returns."""
    gb = _pkg()
    from paper_2311_02909_b200.engine import BulkSampler

    rng = np.random.default_rng(5)
    n, rowptr, col = _rmat(13, 60000, seed=5)
    G = _graph(n, rowptr, col)
    cfg = gb.SamplerConfig.sage(3, 64, (15, 10, 5), bulk_count=4, seed=11)
    jobs = [([rng.permutation(n)[: rng.integers(1, 65)] for _ in range(4)], 4 * j)
            for j in range(5)]
    want = []
    for mode in ("dedup", "pfree"):
        bs = BulkSampler(G, cfg, mode=mode)
        for batches, boff in jobs:
            want.append(bs.sample(batches, epoch=2, batch_offset=boff).to_arrays())
        eps = list(bs.sample_stream(jobs, epoch=2))  # every yielded epoch owns its memory
        got = [ep.to_arrays() for ep in eps]
        assert len(got) == len(jobs)
        for g, w in zip(got, want[-len(jobs):]):
            assert O.compare_epochs(w, g) == []
        # reference types as zero-copy views of the staged arrays
        lay = eps[0].layers[-1]
        assert lay.adjacency.col_indices.base is not None
        assert not lay.adjacency.values.flags.writeable
        assert lay.adjacency.equals(gb.SparseMatrix(*lay.adjacency.shape,
                                                    eps[0].to_arrays()[-1]["adj_ptr"],
                                                    eps[0].to_arrays()[-1]["adj_col"],
                                                    np.ones(lay.adjacency.nnz)))


@pytest.mark.parametrize("mode", MODES)
def test_sage_inclusion_two_thirds(mode):
    """A degree-3 vertex with s = 2 keeps each neighbour with probability 2/3
    (reference test_acceptance.py:80-84), over many minibatches of the
    production Philox stream (distinct keys per batch)."""
    from scipy import stats

    gb = _pkg()
    G = gb.Graph.from_edges(4, [0, 0, 0, 1, 2, 3], [1, 2, 3, 0, 0, 0])
    trials = 30000
    cfg = gb.SamplerConfig.sage(1, 1, (2,), bulk_count=trials, seed=123)
    ep = gb.sample_epoch_bulk(G, cfg, [[0]] * trials, mode=mode)
    a = ep.layers[0].to_arrays()
    cat, off = a["sampv_cat"], a["sampv_off"]
    assert np.all(np.diff(off) == 2)
    counts = np.bincount(cat, minlength=4)[1:]
    assert counts.sum() == 2 * trials
    assert stats.chisquare(counts, f_exp=np.full(3, 2 * trials / 3)).pvalue > 0.01
    pairs = np.bincount((cat.reshape(-1, 2) - 1) @ np.array([3, 1]), minlength=9)
    assert stats.chisquare(pairs[[1, 2, 5]], f_exp=np.full(3, trials / 3)).pvalue > 0.01


def test_sage_per_edge_inclusion_law():
    """Per-edge inclusion min(s, d) / d for every row of a random graph
    (SURVEY.md §8c statistical parity, SAGE): one-layer bulks over many
    epochs, chi-square per vertex on the neighbour counts."""
    from scipy import stats

    gb = _pkg()
    rng = np.random.default_rng(8)
    n, rowptr, col = _rmat(9, 3000, seed=8)
    G = _graph(n, rowptr, col)
    deg = np.diff(rowptr)
    verts = np.flatnonzero((deg > 6) & (deg <= 40))[:24]
    s, epochs = 5, 400
    cfg = gb.SamplerConfig.sage(1, len(verts), (s,), bulk_count=1, seed=3)
    hits = {int(v): np.zeros(deg[v]) for v in verts}
    for e in range(epochs):
        ep = gb.sample_epoch_bulk(G, cfg, [verts], epoch=e, mode="dedup")
        fr = ep.layers[0].frontier
        fp, fc = fr.row_offsets, fr.col_indices
        for i, v in enumerate(verts):
            nb = col[rowptr[v]: rowptr[v + 1]]
            got = fc[fp[i]: fp[i + 1]]
            assert got.size == s
            hits[int(v)][np.searchsorted(nb, got)] += 1
    pv = [stats.chisquare(h, f_exp=np.full(h.size, epochs * s / h.size)).pvalue
          for h in hits.values()]
    # 24 independent tests at 1%: allow one rejection
    assert sum(p < 0.01 for p in pv) <= 1


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("fan", [(40, 3), (7, 100), (33,)])
def test_sage_fanouts_above_32(mode, fan):
    """The reference has no fanout cap (sampler.py:56-66): fanouts above 32
    run the thread-per-row kernel with the sorted picks in the frontier slot;
    bit-exact with the oracle in every mode."""
    gb = _pkg()
    rng = np.random.default_rng(len(fan) + fan[0])
    n, rowptr, col = _rmat(12, 60000, seed=4)
    G = _graph(n, rowptr, col)
    b, k = 48, 4
    batches = [rng.permutation(n)[: rng.integers(1, b + 1)] for _ in range(k)]
    cfg = gb.SamplerConfig.sage(len(fan), b, fan, bulk_count=k, seed=17)
    ep = gb.sample_epoch_bulk(G, cfg, batches, epoch=1, batch_offset=2, mode=mode)
    want = O.sage_bulk(n, rowptr, col, batches, b, fan, 17, 1, 2)
    assert O.compare_epochs(want, ep.to_arrays()) == []


def test_sage_hub_rows_dedup_matches_oracle():
    """Rows longer than the tier-A buffer (hub kernel: chunked TMA staging)
    and rows exactly at the tier boundaries, every mode bit-exact."""
    gb = _pkg()
    rng = np.random.default_rng(77)
    n = 60000
    hubs = {0: 20000, 1: 8192, 2: 8193, 3: 1024, 4: 1025, 5: 70000}
    src, dst = [], []
    for h, d in hubs.items():
        nb = rng.choice(np.arange(6, n), size=min(d, n - 6), replace=False)
        src += [h] * len(nb) + list(nb)
        dst += list(nb) + [h] * len(nb)
    src = np.array(src)
    dst = np.array(dst)
    A = gb.SparseMatrix.from_coo(n, n, src, dst, np.ones(src.size), dedup="first")
    G = gb.Graph(A)
    batches = [np.array([0, 1, 2, 3, 4, 5, 7, 9]), np.arange(6, 300), np.array([5, 5, 0, 1])]
    cfg = gb.SamplerConfig.sage(3, 300, (15, 10, 5), bulk_count=3, seed=2)
    want = O.sage_bulk(n, A.row_offsets, A.col_indices, batches, 300, (15, 10, 5), 2, 0, 0)
    for mode in MODES:
        ep = gb.sample_epoch_bulk(G, cfg, batches, mode=mode)
        assert O.compare_epochs(want, ep.to_arrays()) == [], mode


def _baseline_graph(shape):
    gb = _pkg()
    from paper_2311_02909_b200.graphgen import SHAPES, rmat_device_graph

    n, m, sym = SHAPES[shape]
    dg = rmat_device_graph(n, m, symmetric=sym, seed=0)
    return gb.Graph.from_device(dg), dg


def _baseline_batches(n, k):
    from paper_2311_02909_b200.pipeline import make_batches

    return make_batches(np.arange(n), 1024, seed=0, epoch=0)[:k]


@pytest.mark.parametrize("mode", MODES)
def test_cfg1_bulk_matches_oracle(mode):
    """BASELINE configs[0] exactly: R-MAT scale 16 (65,536 vertices, 2^20
    undirected pairs), b = 1024, (15, 10, 5), k = 8 — bit-exact with the C
    oracle (which is pinned to the reference's own outputs)."""
    G, dg = _baseline_graph("cfg1")
    batches = _baseline_batches(dg.n, 8)
    cfg = _pkg().SamplerConfig.sage(3, 1024, (15, 10, 5), bulk_count=8, seed=0)
    ep = _pkg().sample_epoch_bulk(G, cfg, batches, mode=mode)
    rowptr = dg.rowptr.cpu().numpy()
    col = dg.col[: dg.nnz].cpu().numpy()
    want = O.sage_bulk(dg.n, rowptr, col, batches, 1024, (15, 10, 5), 0, 0, 0, threads=8)
    assert O.compare_epochs(want, ep.to_arrays()) == []


def test_cfg2_full_size_bulk_matches_oracle():
    """BASELINE configs[1] at full size: products-shape R-MAT (2,449,029
    vertices, 123.7M entries), b = 1024, (15, 10, 5), k = 64 through the
    bench's engine path (SageBulk, dedup Alg. 1) — every layer bit-exact with
    the C oracle on all 64 minibatches."""
    import torch

    from paper_2311_02909_b200.engine import SageBulk, upload_batches

    G, dg = _baseline_graph("products")
    batches = _baseline_batches(dg.n, 64)
    d_off, d_cat, r1 = upload_batches(batches, dg.n, 1024)
    bulk = SageBulk(dg, 64, r1, 1024, (15, 10, 5), mode="dedup")
    bulk.launch(d_off, d_cat, 0, 0, 0)
    torch.cuda.synchronize()
    from paper_2311_02909_b200.sampler import SampledEpoch, SamplerKind

    got = SampledEpoch(SamplerKind.SAGE, 0, batches, bulk.layers(d_off, d_cat), 3).to_arrays()
    rowptr = dg.rowptr.cpu().numpy()
    col = dg.col[: dg.nnz].cpu().numpy()
    want = O.sage_bulk(dg.n, rowptr, col, batches, 1024, (15, 10, 5), 0, 0, 0,
                       threads=os.cpu_count() or 8)
    assert O.compare_epochs(want, got) == []


def test_sage_bulks_on_recycled_memory():
    """Workspace memory recycled by the caching allocator between bulks
    (other tensors written into it, as run_epoch's feature arrays do) must
    not leak stale counters or bit maps into the next bulk: a sequence of
    small bulks, each followed by dirtying allocations, every one bit-exact
    (the reference test_acceptance test_09 sequence that exposed it)."""
    import torch

    gb = _pkg()
    rng = np.random.default_rng(9)
    n, d, b = 230, 5, 7
    src = np.repeat(np.arange(n), d)
    dst = np.concatenate([rng.choice(np.delete(np.arange(n), v), d, replace=False)
                         for v in range(n)])
    G = gb.Graph.from_edges(n, src, dst)
    A = G.adjacency
    cfg = gb.SamplerConfig.sage(2, b, (3, 2), bulk_count=1, seed=19)
    for boff in range(24):
        batches = [] if boff % 3 == 2 else [rng.permutation(n)[:b]]
        ep = gb.sample_epoch_bulk(G, cfg, batches, batch_offset=boff, mode="dedup")
        if batches:
            want = O.sage_bulk(n, A.row_offsets, A.col_indices, batches, b, (3, 2), 19, 0, boff)
            assert O.compare_epochs(want, ep.to_arrays()) == [], boff
        del ep
        junk = [torch.full((4096 * (i + 1),), 7, dtype=torch.int32, device="cuda")
                for i in range(6)]
        del junk


@pytest.mark.parametrize("mode", MODES)
def test_sparse_extraction_forced_matches_oracle(mode, monkeypatch):
    """The touched-record extraction (k_touch / k_rec_scan_touch /
    k_enum_touch, the default for n >= 2^23) forced on small graphs: random
    cases, hub rows and several fanout buckets bit-exact with the oracle,
    then the dense extraction again on the same (clean) workspace."""
    gb = _pkg()
    monkeypatch.setenv("GB_SPARSE_EXTRACT", "1")
    for case in range(3):
        rng = np.random.default_rng(300 + case)
        n, rowptr, col = _rmat(12 + case % 2, 30000 * (1 + case), seed=case + 11)
        G = _graph(n, rowptr, col)
        b, k = [40, 128, 300][case], [2, 7, 4][case]
        fan = [(15, 10, 5), (3, 2), (25, 1, 8)][case]
        batches = [rng.permutation(n)[: rng.integers(1, b + 1)] for _ in range(k)]
        cfg = gb.SamplerConfig.sage(len(fan), b, fan, bulk_count=k, seed=case + 5)
        want = O.sage_bulk(n, rowptr, col, batches, b, fan, case + 5, 1, 2)
        ep = gb.sample_epoch_bulk(G, cfg, batches, epoch=1, batch_offset=2, mode=mode)
        assert O.compare_epochs(want, ep.to_arrays()) == [], case
        monkeypatch.setenv("GB_SPARSE_EXTRACT", "0")
        ep = gb.sample_epoch_bulk(G, cfg, batches, epoch=1, batch_offset=2, mode=mode)
        assert O.compare_epochs(want, ep.to_arrays()) == [], case
        monkeypatch.setenv("GB_SPARSE_EXTRACT", "1")


def test_sparse_extraction_default_on_large_n():
    """n >= 2^23 takes the touched-record extraction by default: a sparse
    random graph over 2^23 + 5 vertices, k = 6, bit-exact with the oracle."""
    gb = _pkg()
    rng = np.random.default_rng(9)
    n = (1 << 23) + 5
    m = 600000
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    hub = rng.integers(0, n, 20)
    src = np.concatenate([src, np.repeat(hub, 3000), rng.integers(0, n, 60000)])
    dst = np.concatenate([dst, rng.integers(0, n, 60000), np.repeat(hub, 3000)])
    G = gb.Graph.from_edges(n, np.concatenate([src, dst]), np.concatenate([dst, src]))
    A = G.adjacency
    batches = [np.concatenate([hub[:5], rng.integers(0, n, 200)]) for _ in range(6)]
    batches = [np.unique(x) for x in batches]
    cfg = gb.SamplerConfig.sage(3, 256, (15, 10, 5), bulk_count=6, seed=4)
    want = O.sage_bulk(n, A.row_offsets, A.col_indices, batches, 256, (15, 10, 5), 4, 0, 0)
    for mode in MODES:
        ep = gb.sample_epoch_bulk(G, cfg, batches, mode=mode)
        assert O.compare_epochs(want, ep.to_arrays()) == [], mode


def test_grouped_path_forced_everywhere(monkeypatch):
    """The dedup bulk's grouped path (count / items / rows / pick / serve
    tiers) forced on every layer — including layers the default rule samples
    P-free — on random cases and the hub-row graph, with everything staged
    and with everything direct: bit-exact with the oracle."""
    gb = _pkg()
    monkeypatch.setenv("GB_DEDUP_FROM", "0")
    monkeypatch.setenv("GB_GROUP_RATIO", "0")
    for case in range(3):
        rng = np.random.default_rng(500 + case)
        n, rowptr, col = _rmat(12 + case % 2, 30000 * (1 + case), seed=case + 21)
        G = _graph(n, rowptr, col)
        b, k = [40, 128, 300][case], [2, 7, 4][case]
        fan = [(15, 10, 5), (3, 2), (25, 1, 8)][case]
        batches = [rng.permutation(n)[: rng.integers(1, b + 1)] for _ in range(k)]
        cfg = gb.SamplerConfig.sage(len(fan), b, fan, bulk_count=k, seed=case + 9)
        want = O.sage_bulk(n, rowptr, col, batches, b, fan, case + 9, 2, 1)
        for ratio in ("0", "1"):  # every row staged / direct wherever picks < 8 d
            monkeypatch.setenv("GB_DIRECT_RATIO", ratio)
            ep = gb.sample_epoch_bulk(G, cfg, batches, epoch=2, batch_offset=1, mode="dedup")
            assert O.compare_epochs(want, ep.to_arrays()) == [], (case, ratio)
