"""Generate the golden fixtures that pin the oracle and the CUDA sampler.

Run HERE (the container that has /root/reference); the outputs are small
.npz files committed next to this script, so the GPU box never needs the
reference:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture is produced by the UNMODIFIED reference package
(`/root/reference/pkg/src/gnnbulk`) with one substitution: the per-row
random stream `RowRng.stream` (`sampler.py:112-116`) is replaced by the
counter-based uniform source of `oracle/philox.py`, exactly as SURVEY.md
§8(c)(i) prescribes, so that the CUDA sampler (which draws the same
uniforms on the device) must reproduce the reference output bit for bit.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import gnnbulk  # noqa: E402  (the reference)
from gnnbulk import sampler as ref_sampler  # noqa: E402
from gnnbulk.sparse import Graph, SparseMatrix  # noqa: E402

from oracle.philox import InjectedStream  # noqa: E402


def patch_rng():
    def stream(self, global_row):
        return InjectedStream(self.seed, self.epoch, self.layer, global_row)

    ref_sampler.RowRng.stream = stream


# -- graphs -----------------------------------------------------------------


def rmat_edges(scale, m_target, seed, a=0.57, b=0.19, c=0.19, n=None):
    """Graph500-style R-MAT, rejecting ids >= n and self loops, keeping the
    first m_target unique undirected pairs, randomly relabelled
    (SURVEY.md Appendix B recipe, reduced sizes)."""
    rng = np.random.default_rng(seed)
    n = n or (1 << scale)
    got = set()
    pairs = []
    while len(pairs) < m_target:
        cnt = 4 * m_target
        u = np.zeros(cnt, dtype=np.int64)
        v = np.zeros(cnt, dtype=np.int64)
        for lvl in range(scale):
            r = rng.random(cnt)
            bit_u = r >= a + b
            bit_v = ((r >= a) & (r < a + b)) | (r >= a + b + c)
            u |= bit_u.astype(np.int64) << lvl
            v |= bit_v.astype(np.int64) << lvl
        for x, y in zip(u.tolist(), v.tolist()):
            if x >= n or y >= n or x == y:
                continue
            key = (min(x, y), max(x, y))
            if key in got:
                continue
            got.add(key)
            pairs.append(key)
            if len(pairs) == m_target:
                break
    perm = rng.permutation(n)
    e = np.array(pairs, dtype=np.int64)
    src = perm[e[:, 0]]
    dst = perm[e[:, 1]]
    return n, np.concatenate([src, dst]), np.concatenate([dst, src])


def figure_graph():
    edges = [(0, 1), (1, 4), (2, 5), (3, 5), (4, 5)]
    src = [u for u, v in edges] + [v for u, v in edges]
    dst = [v for u, v in edges] + [u for u, v in edges]
    return 6, np.array(src), np.array(dst)


def hub_graph(seed):
    """A few hubs with degrees spanning 1..6000 plus a sparse background, to
    exercise every binade of the exact SAGE replay table."""
    rng = np.random.default_rng(seed)
    n = 8000
    src, dst = [], []
    for h, d in enumerate([1, 2, 3, 15, 16, 17, 100, 1023, 1024, 1025, 3000, 5999]):
        nb = rng.choice(np.arange(12, n), size=d, replace=False)
        src += [h] * d
        dst += nb.tolist()
    bg = rng.integers(12, n, size=(6 * n, 2))
    src += bg[:, 0].tolist()
    dst += bg[:, 1].tolist()
    src, dst = np.array(src), np.array(dst)
    return n, np.concatenate([src, dst]), np.concatenate([dst, src])


# -- serialisation --------------------------------------------------------


def pack_csr(prefix, M: SparseMatrix, out, values=True):
    out[prefix + "_shape"] = np.array(M.shape, dtype=np.int64)
    out[prefix + "_ptr"] = np.asarray(M.row_offsets, dtype=np.int64)
    out[prefix + "_col"] = np.asarray(M.col_indices, dtype=np.int64)
    if values:
        out[prefix + "_val"] = np.asarray(M.values, dtype=np.float64)


def pack_ragged(prefix, arrays, out):
    arrays = [np.asarray(a, dtype=np.int64) for a in arrays]
    off = np.zeros(len(arrays) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(a) for a in arrays])
    out[prefix + "_off"] = off
    out[prefix + "_cat"] = np.concatenate(arrays) if arrays else np.zeros(0, np.int64)


def pack_epoch(ep, out):
    out["kind"] = np.array(str(ep.kind.value))
    out["n_layers"] = np.array(len(ep.layers))
    out["spgemm_calls"] = np.array(ep.spgemm_calls)
    for li, layer in enumerate(ep.layers):
        p = f"L{li}"
        assert np.all(layer.frontier.values == 1.0)
        assert np.all(layer.adjacency.values == 1.0)
        pack_csr(p + "_frontier", layer.frontier, out, values=False)
        pack_csr(p + "_adj", layer.adjacency, out, values=False)
        pack_ragged(p + "_rowv", layer.row_vertices, out)
        pack_ragged(p + "_colv", layer.col_vertices, out)
        pack_ragged(p + "_sampv", layer.sampled_vertices, out)


def epoch_case(name, graph, kind, layers, b, fanouts, k, seed, epoch=0,
               batch_offset=0, batch_seed=0):
    n, src, dst = graph
    G = Graph.from_edges(n, src, dst)
    rng = np.random.default_rng(batch_seed)
    if isinstance(k, list):
        batches = [np.asarray(x, dtype=np.int64) for x in k]
    else:
        batches = [rng.permutation(n)[:b] for _ in range(k)]
    if kind == "sage":
        cfg = gnnbulk.SamplerConfig.sage(layers, b, fanouts, bulk_count=len(batches), seed=seed)
    else:
        cfg = gnnbulk.SamplerConfig.ladies(layers, b, fanouts, bulk_count=len(batches), seed=seed)
    ep = gnnbulk.sample_epoch_bulk(G, cfg, batches, epoch=epoch, batch_offset=batch_offset)
    out = {}
    pack_csr("A", G.adjacency, out, values=False)
    pack_ragged("batches", batches, out)
    out["cfg"] = np.array([layers, b, seed, epoch, batch_offset], dtype=np.int64)
    out["fanouts"] = np.array(cfg.fanouts, dtype=np.int64)
    pack_epoch(ep, out)
    np.savez_compressed(os.path.join(HERE, f"epoch_{name}.npz"), **out)
    sizes = [(l.frontier.n_rows, l.frontier.nnz, l.adjacency.n_cols) for l in ep.layers]
    print(f"epoch_{name}: n={n} nnz={G.adjacency.nnz} layers={sizes}")


def its_cases():
    """its_sample_row (sampler.py:157-189) with explicit uniforms, including
    the u -> 1^- clamp, for the SAGE replay table and the generic path."""

    class ListRng:
        def __init__(self, us):
            self.us = list(us)

        def random(self):
            return self.us.pop(0)

    rng = np.random.default_rng(7)
    degs, fans, us, picks = [], [], [], []
    weights_cat, weights_off = [], [0]
    kinds = []
    top = 1.0 - 2.0 ** -53
    for case in range(3000):
        if case < 1500:
            m = int(rng.integers(1, 400)) if case % 5 else int(rng.integers(400, 20000))
            s = int(rng.integers(1, 20))
            w = np.full(m, 1.0) / m  # what norm_rows_sage produces: fl(1/deg)
            kinds.append(0)
        else:
            m = int(rng.integers(1, 300))
            s = int(rng.integers(1, 40))
            cnt = rng.integers(1, 20, size=m).astype(np.float64)
            w = (cnt * cnt) / np.sum(cnt * cnt)  # norm_rows_ladies: e^2/sum e^2
            kinds.append(1)
        take = min(s, m)
        u = rng.random(max(take, 1))
        if case % 7 == 0:
            u[rng.integers(0, len(u))] = top
        if case % 11 == 0:
            u[:] = 0.0
        p = ref_sampler.its_sample_row(w, s, ListRng(u.tolist()))
        degs.append(m)
        fans.append(s)
        us.append(np.pad(u, (0, 40 - len(u))))
        picks.append(np.pad(p, (0, 40 - len(p)), constant_values=-1))
        weights_cat.append(w)
        weights_off.append(weights_off[-1] + m)
    np.savez_compressed(
        os.path.join(HERE, "its_rows.npz"),
        deg=np.array(degs), fanout=np.array(fans), kind=np.array(kinds),
        u=np.array(us), picks=np.array(picks),
        w_cat=np.concatenate(weights_cat), w_off=np.array(weights_off),
    )
    print("its_rows: 3000 rows")


def spgemm_cases():
    """spgemm/norm goldens from the reference (scipy csr_matmat order) on
    non-dyadic values, so accumulation order is pinned bit for bit."""
    rng = np.random.default_rng(9)
    out = {}
    for i in range(40):
        m, kk, nn = (int(x) for x in rng.integers(1, 70, size=3))
        dens = float(rng.uniform(0.02, 0.5))
        A = SparseMatrix.from_dense(
            np.where(rng.random((m, kk)) < dens, rng.random((m, kk)) * 3 - 1, 0.0))
        B = SparseMatrix.from_dense(
            np.where(rng.random((kk, nn)) < dens, rng.random((kk, nn)) * 3 - 1, 0.0))
        C = gnnbulk.spgemm(A, B)
        pack_csr(f"c{i}_A", A, out)
        pack_csr(f"c{i}_B", B, out)
        pack_csr(f"c{i}_C", C, out)
        Pos = SparseMatrix(C.n_rows, C.n_cols, C.row_offsets, C.col_indices,
                           np.abs(C.values) + 0.25, validate=False)
        pack_csr(f"c{i}_P", Pos, out)
        pack_csr(f"c{i}_NS", gnnbulk.norm_rows_sage(Pos), out)
        pack_csr(f"c{i}_NL", gnnbulk.norm_rows_ladies(Pos), out)
    out["count"] = np.array(40)
    np.savez_compressed(os.path.join(HERE, "spgemm.npz"), **out)
    print("spgemm: 40 cases")


def pipeline_cases():
    """The reference's epoch pipeline (pipeline.py:78-130, 200-305) on the
    injected-uniform epochs: per-batch fetch_features + _propagate_batch
    outputs (float64) for SAGE and LADIES bulks, fetch_features on a 4 x 2
    grid with its ledger, and run_epoch's accounting on three grids."""
    from gnnbulk import pipeline as ref_pipeline
    from gnnbulk.dist import CommLedger, ProcessGrid

    n, src, dst = rmat_edges(10, 6000, seed=1)
    G = Graph.from_edges(n, src, dst)
    H = gnnbulk.synthesize_features(n, 8, 5)
    out = {}
    pack_csr("A", G.adjacency, out, values=False)
    out["H"] = H
    rng = np.random.default_rng(12)
    for kind in ("sage", "ladies"):
        if kind == "sage":
            cfg = gnnbulk.SamplerConfig.sage(3, 16, (6, 4, 3), bulk_count=4, seed=3)
            batches = [rng.permutation(n)[: rng.integers(1, 17)] for _ in range(4)]
        else:
            cfg = gnnbulk.SamplerConfig.ladies(2, 16, 12, bulk_count=4, seed=3)
            batches = [np.sort(rng.permutation(n)[: rng.integers(1, 17)]) for _ in range(4)]
        ep = gnnbulk.sample_epoch_bulk(G, cfg, batches, epoch=2, batch_offset=3)
        grid = ProcessGrid(1, 1)
        Hp = ref_pipeline.FeaturePartition.partition(H, grid)
        ys = []
        for b in range(len(batches)):
            X = ref_pipeline.fetch_features(ep.layers[-1].col_vertices[b], Hp, grid)
            ys.append(ref_pipeline._propagate_batch(ep, b, X))
        pack_ragged(f"{kind}_batches", batches, out)
        out[f"{kind}_cfg"] = np.array([cfg.layers, cfg.batch_size, cfg.seed] + list(cfg.fanouts),
                                      dtype=np.int64)
        out[f"{kind}_Y"] = np.concatenate(ys)
        out[f"{kind}_Yoff"] = np.cumsum([0] + [y.shape[0] for y in ys])
        sub = {}
        pack_epoch(ep, sub)
        for key, val in sub.items():
            out[f"{kind}_ep_{key}"] = val
    grid = ProcessGrid(4, 2)
    Hp = ref_pipeline.FeaturePartition.partition(H, grid)
    verts = rng.integers(0, n, size=400)
    out["fetch_verts"] = verts
    words = np.zeros((4, 4), dtype=np.int64)  # requester x process
    msgs = np.zeros((4, 4), dtype=np.int64)
    for req in range(4):
        led = CommLedger(4)
        rows = ref_pipeline.fetch_features(verts, Hp, grid, led, req)
        assert np.array_equal(rows, H[verts])
        for proc in range(4):
            words[req, proc] = led.words(phase="all-to-allv", process=proc)
            msgs[req, proc] = led.messages(phase="all-to-allv", process=proc)
    out["fetch_words"], out["fetch_msgs"] = words, msgs
    cfg = gnnbulk.SamplerConfig.sage(2, 64, (5, 3), bulk_count=4, seed=6)
    acc = []
    for p, c, mode in ((1, 1, "replicated"), (4, 1, "replicated"), (4, 2, "partitioned")):
        grid = ProcessGrid(p, c)
        rep = ref_pipeline.run_epoch(G, ref_pipeline.FeaturePartition.partition(H, grid), cfg,
                                     grid, mode=mode, epoch=1)
        led = rep.ledger
        row = [p, c, rep.n_batches, rep.chunks, rep.spgemm_calls]
        row += list(rep.batches_per_process) + [0] * (4 - p)
        row += [led.messages(phase=ph) for ph in gnnbulk.PHASES]
        row += [led.words(phase=ph) for ph in gnnbulk.PHASES]
        acc.append(row)
    out["run_epoch"] = np.array(acc, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "pipeline.npz"), **out)
    print("pipeline: propagate (sage, ladies), fetch 4x2, run_epoch x3")


def main():
    patch_rng()
    fig = figure_graph()
    epoch_case("fig_sage", fig, "sage", 2, 2, (2, 2), [[1, 5]], seed=3)
    epoch_case("fig_ladies", fig, "ladies", 2, 2, 2, [[1, 5], [0, 2, 3]], seed=3)
    small = rmat_edges(10, 6000, seed=1)
    epoch_case("rmat10_sage", small, "sage", 3, 16, (15, 10, 5), 4, seed=5, batch_seed=2)
    epoch_case("rmat10_sage_off", small, "sage", 2, 8, (4, 3), 5, seed=11, epoch=3,
               batch_offset=17, batch_seed=4)
    epoch_case("rmat10_ladies", small, "ladies", 3, 8, 6, 3, seed=5, batch_seed=3)
    epoch_case("rmat10_ladies_clamp", small, "ladies", 2, 3, 40, 4, seed=8, batch_seed=5)
    hubs = hub_graph(3)
    epoch_case("hubs_sage", hubs, "sage", 2, 12, (20, 7), [list(range(12)), [0, 5, 11, 40]],
               seed=2)
    mid = rmat_edges(12, 40000, seed=6)
    epoch_case("rmat12_sage", mid, "sage", 3, 64, (15, 10, 5), 4, seed=0, batch_seed=6)
    epoch_case("rmat12_ladies", mid, "ladies", 2, 64, 32, 3, seed=0, batch_seed=7)
    its_cases()
    spgemm_cases()
    pipeline_cases()


if __name__ == "__main__":
    main()
