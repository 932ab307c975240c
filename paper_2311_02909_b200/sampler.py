"""Bulk minibatch samplers (GraphSAGE node-wise, LADIES layer-wise) on B200.

Host-side mirror of the reference sampler API
(`pkg/src/gnnbulk/sampler.py`): same names, argument meaning and error
behaviour.  The per-layer work — P = Q^l A, normalisation, keyed
inverse-transform sampling and extraction — runs in the CUDA library
(`csrc/`, C ABI `include/gnnbulk_b200.h`) for all k stacked minibatches at
once; results stay in HBM (`LayerSample.device`) and are converted to the
reference's host types only when a host field is read.

Randomness: one counter-based stream per (seed, epoch, layer, global_row),
u(seed, epoch, layer, row, t) = Philox4x64-10 (see gb_common.cuh), so bulk,
per-batch, chunked and distributed runs draw identical samples
(the reference's keyed-stream contract, sampler.py:9-11, 97-116).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import ContractViolation
from .sparse import Graph, SparseMatrix


class SamplerKind(str, Enum):
    SAGE = "sage"
    LADIES = "ladies"


@dataclass(frozen=True)
class SamplerConfig:
    """Hyperparameters of a sampling run (reference sampler.py:41-94).

    fanouts: per-layer sample count, outermost layer first; for layer-wise
    sampling every entry is the layer width s.
    """

    kind: SamplerKind
    layers: int
    batch_size: int
    fanouts: tuple
    bulk_count: int
    seed: int

    def __post_init__(self):
        if self.layers < 1:
            raise ContractViolation("layers must be >= 1")
        if self.batch_size < 1:
            raise ContractViolation("batch_size must be >= 1")
        if self.bulk_count < 1:
            raise ContractViolation("bulk_count must be >= 1")
        if len(self.fanouts) != self.layers:
            raise ContractViolation("fanouts must have one entry per layer")
        if any(int(s) < 1 for s in self.fanouts):
            raise ContractViolation("fanouts must be >= 1")
        object.__setattr__(self, "kind", SamplerKind(self.kind))
        object.__setattr__(self, "fanouts", tuple(int(s) for s in self.fanouts))

    @classmethod
    def sage(cls, layers, batch_size, fanouts, bulk_count=1, seed=0):
        if isinstance(fanouts, int):
            fanouts = (fanouts,) * layers
        return cls(SamplerKind.SAGE, layers, batch_size, tuple(fanouts), bulk_count, seed)

    @classmethod
    def ladies(cls, layers, batch_size, sample_num, bulk_count=1, seed=0):
        return cls(SamplerKind.LADIES, layers, batch_size, (sample_num,) * layers,
                   bulk_count, seed)

    @property
    def s(self):
        return self.fanouts[0]

    def rows_per_batch(self, depth):
        """Nominal rows one batch contributes at `depth` (1-based): the stride
        of the global row keys."""
        if self.kind is SamplerKind.LADIES:
            return 1
        rows = self.batch_size
        for s in self.fanouts[: depth - 1]:
            rows *= s
        return rows


class KeyedStream:
    """Stream of one row: the t-th `.random()` is u(seed, epoch, layer, row, t),
    drawn on the device (gb_uniforms)."""

    __slots__ = ("seed", "epoch", "layer", "row", "t")

    def __init__(self, seed, epoch, layer, row):
        self.seed, self.epoch, self.layer, self.row = int(seed), int(epoch), int(layer), int(row)
        self.t = 0

    def random(self, size=None):
        from . import ops

        n = 1 if size is None else int(size)
        u = ops.uniforms(self.seed, self.epoch, self.layer,
                         np.full(n, self.row, dtype=np.int64),
                         np.arange(self.t, self.t + n, dtype=np.int64))
        self.t += n
        return float(u[0]) if size is None else u


class RowRng:
    """Deterministic per-row streams keyed by (seed, epoch, layer, global_row)
    (reference sampler.py:97-116)."""

    __slots__ = ("seed", "epoch", "layer")

    def __init__(self, seed, epoch, layer):
        self.seed = int(seed)
        self.epoch = int(epoch)
        self.layer = int(layer)

    def stream(self, global_row) -> KeyedStream:
        return KeyedStream(self.seed, self.epoch, self.layer, global_row)


# -- seed matrices (sampler.py:122-151) ------------------------------------------


def _flatten_batches(batches, n, sort_within=False):
    arrs, offsets = [], np.zeros(len(batches) + 1, dtype=np.int64)
    for i, batch in enumerate(batches):
        ids = np.asarray(batch, dtype=np.int64).ravel()
        if ids.size and (ids.min() < 0 or ids.max() >= n):
            raise ContractViolation("batch vertex id out of range")
        if sort_within:
            ids = np.sort(ids)
            if ids.size > 1 and np.any(ids[1:] == ids[:-1]):
                raise ContractViolation("batch vertices must be distinct")
        arrs.append(ids)
        offsets[i + 1] = offsets[i] + ids.size
    cat = np.concatenate(arrs) if arrs else np.zeros(0, dtype=np.int64)
    return cat, offsets


def sage_seed_matrix(batches, n) -> SparseMatrix:
    """One one-hot row per batch vertex, batches stacked in order."""
    cols, _ = _flatten_batches(batches, n)
    m = cols.size
    return SparseMatrix(m, n, np.arange(m + 1), cols, np.ones(m), validate=False)


def ladies_seed_matrix(batches, n) -> SparseMatrix:
    """One row per batch with a 1 at every (sorted, distinct) batch vertex."""
    cols, offsets = _flatten_batches(batches, n, sort_within=True)
    return SparseMatrix(len(batches), n, offsets, cols, np.ones(cols.size))


# -- epoch-level results (sampler.py:240-306) -------------------------------------


def _split(cat, off):
    return tuple(cat[off[i]:off[i + 1]].copy() for i in range(len(off) - 1))


def _views(cat, off):
    out = []
    for i in range(len(off) - 1):
        v = cat[int(off[i]):int(off[i + 1])]
        v.setflags(write=False)
        out.append(v)
    return tuple(out)


class LayerSample:
    """Sampling output of one layer (reference sampler.py:240-261).

    Results produced on the device keep their tensors in `.device` (a dict of
    torch tensors, flat CSR arrays + per-batch offsets) and build the
    reference host fields (`frontier`, `adjacency`, `row_vertices`,
    `col_vertices`, `sampled_vertices`) lazily on first access.
    """

    def __init__(self, depth, frontier=None, adjacency=None, row_vertices=None,
                 col_vertices=None, sampled_vertices=None, device=None, n=None):
        self.depth = int(depth)
        self.device = device
        self._n = n
        self._host = None
        if device is None:
            self._host = {
                "frontier": frontier, "adjacency": adjacency,
                "row_vertices": tuple(row_vertices), "col_vertices": tuple(col_vertices),
                "sampled_vertices": tuple(sampled_vertices),
            }

    # flat host arrays in the oracle's format (oracle/oracle.py LAYER_KEYS)
    def to_arrays(self):
        if self.device is not None:
            d = {k: (v if isinstance(v, np.ndarray) else v.cpu().numpy()).astype(np.int64)
                 for k, v in self.device.items() if k not in ("frontier_shape", "adj_shape")}
            d["frontier_shape"] = np.asarray(self.device["frontier_shape"], dtype=np.int64)
            d["adj_shape"] = np.asarray(self.device["adj_shape"], dtype=np.int64)
            return d
        h = self._host

        def rag(arrs):
            off = np.zeros(len(arrs) + 1, dtype=np.int64)
            off[1:] = np.cumsum([len(a) for a in arrs])
            cat = np.concatenate([np.asarray(a, np.int64) for a in arrs]) if arrs else \
                np.zeros(0, np.int64)
            return off, cat

        out = {}
        for name, M in (("frontier", h["frontier"]), ("adj", h["adjacency"])):
            out[name + "_shape"] = np.array(M.shape, dtype=np.int64)
            out[name + "_ptr"] = M.row_offsets.astype(np.int64)
            out[name + "_col"] = M.col_indices.astype(np.int64)
        for name, key in (("rowv", "row_vertices"), ("colv", "col_vertices"),
                          ("sampv", "sampled_vertices")):
            out[name + "_off"], out[name + "_cat"] = rag(h[key])
        return out

    def _materialise(self):
        if self._host is None and self.device is not None and all(
                isinstance(v, (np.ndarray, tuple)) for v in self.device.values()):
            # host-staged flat arrays (BulkSampler): reference types as
            # zero-copy views — CSR over the staged offsets / columns, the
            # per-batch tuples as slices of the concatenated arrays
            d = self.device
            fs, ads = d["frontier_shape"], d["adj_shape"]
            self._host = {
                "frontier": SparseMatrix.trusted(fs[0], fs[1], d["frontier_ptr"],
                                                 d["frontier_col"]),
                "adjacency": SparseMatrix.trusted(ads[0], ads[1], d["adj_ptr"], d["adj_col"]),
                "row_vertices": _views(d["rowv_cat"], d["rowv_off"]),
                "col_vertices": _views(d["colv_cat"], d["colv_off"]),
                "sampled_vertices": _views(d["sampv_cat"], d["sampv_off"]),
            }
        if self._host is None:
            a = self.to_arrays()
            fs, ads = a["frontier_shape"], a["adj_shape"]
            F = a["frontier_col"].size
            A = a["adj_col"].size
            self._host = {
                "frontier": SparseMatrix(fs[0], fs[1], a["frontier_ptr"], a["frontier_col"],
                                         np.ones(F), validate=False),
                "adjacency": SparseMatrix(ads[0], ads[1], a["adj_ptr"], a["adj_col"],
                                          np.ones(A), validate=False),
                "row_vertices": _split(a["rowv_cat"], a["rowv_off"]),
                "col_vertices": _split(a["colv_cat"], a["colv_off"]),
                "sampled_vertices": _split(a["sampv_cat"], a["sampv_off"]),
            }
        return self._host

    @property
    def frontier(self):
        return self._materialise()["frontier"]

    @property
    def adjacency(self):
        return self._materialise()["adjacency"]

    @property
    def row_vertices(self):
        return self._materialise()["row_vertices"]

    @property
    def col_vertices(self):
        return self._materialise()["col_vertices"]

    @property
    def sampled_vertices(self):
        return self._materialise()["sampled_vertices"]

    def frontier_size(self):
        if self.device is not None:
            return int(self.device["frontier_col"].numel())
        return int(sum(len(v) for v in self.sampled_vertices))

    def batch_row_counts(self):
        return [len(v) for v in self.row_vertices]


class SampledEpoch:
    """All layers of sampled structure for a set of minibatches
    (reference sampler.py:264-306)."""

    def __init__(self, kind, epoch, batches, layers, spgemm_calls):
        self.kind = SamplerKind(kind)
        self.epoch = int(epoch)
        self.batches = tuple(batches)
        self.layers = tuple(layers)
        self.spgemm_calls = int(spgemm_calls)

    def deepest_frontier(self, batch_index):
        return self.layers[-1].sampled_vertices[batch_index]

    def to_arrays(self):
        return [layer.to_arrays() for layer in self.layers]

    def equals(self, other) -> bool:
        if (self.kind != other.kind or self.epoch != other.epoch
                or len(self.batches) != len(other.batches)
                or len(self.layers) != len(other.layers)):
            return False
        if any(not np.array_equal(a, b) for a, b in zip(self.batches, other.batches)):
            return False
        for la, lb in zip(self.layers, other.layers):
            if la.depth != lb.depth:
                return False
            a, b = la.to_arrays(), lb.to_arrays()
            for key in a:
                if not np.array_equal(a[key], b[key]):
                    return False
        return True


def sage_batch_blocks(frontier, row_starts):
    """Per-batch node-wise extraction pieces (reference sampler.py:390-406):
    compacted blocks, global column ids, sampled vertices in row order."""
    from . import ops

    blocks, col_maps, new_rows = [], [], []
    for i in range(len(row_starts) - 1):
        block = frontier.row_slice(int(row_starts[i]), int(row_starts[i + 1]))
        compacted, col_map = ops.compact_columns(block)
        blocks.append(compacted)
        col_maps.append(col_map)
        new_rows.append(np.asarray(block.col_indices).copy())
    return blocks, col_maps, new_rows


def build_sage_layer(depth, frontier, blocks, col_maps, row_vertices, new_rows):
    from . import ops

    return LayerSample(depth, frontier, ops.block_diag(blocks),
                       tuple(np.asarray(v).copy() for v in row_vertices), tuple(col_maps),
                       tuple(new_rows))


def ladies_assemble(ar_blocks, qc_blocks):
    """Layer-wise extraction (reference sampler.py:420-434): shared columns
    when every batch sampled the same count, else per-batch diagonal blocks."""
    from . import ops

    if not qc_blocks:
        return SparseMatrix.empty(0, 0)
    if len({b.n_cols for b in qc_blocks}) == 1:
        return ops.spgemm(ops.block_diag(ar_blocks), ops.vstack(qc_blocks))
    return ops.block_diag([ops.spgemm(a, q) for a, q in zip(ar_blocks, qc_blocks)])


def ladies_batch_blocks(Q, frontier, AR, n):
    """Per-batch layer-wise extraction pieces (reference sampler.py:437-451)."""
    from . import ops

    ar_starts = np.concatenate([[0], np.cumsum(Q.row_nnz())])
    sampled, qc_blocks, ar_blocks = [], [], []
    for i in range(Q.n_rows):
        cols = frontier.row_cols(i)
        sampled.append(np.asarray(cols).copy())
        qc_blocks.append(ops.build_column_extraction(cols, n))
        ar_blocks.append(AR.row_slice(int(ar_starts[i]), int(ar_starts[i + 1])))
    return ar_blocks, qc_blocks, sampled


def build_ladies_layer(depth, frontier, adjacency, row_vertices, sampled):
    return LayerSample(depth, frontier, adjacency,
                       tuple(np.asarray(v).copy() for v in row_vertices),
                       tuple(np.asarray(s).copy() for s in sampled),
                       tuple(np.asarray(s).copy() for s in sampled))


def global_row_keys(cfg: SamplerConfig, depth, batch_ids, rows_per_batch_actual):
    """Global row ids of stacked per-batch rows (reference sampler.py:309-322)."""
    stride = cfg.rows_per_batch(depth)
    keys = []
    for b, actual in zip(batch_ids, rows_per_batch_actual):
        if actual > stride:
            raise ContractViolation("actual rows exceed the nominal stride")
        keys.append(b * stride + np.arange(actual, dtype=np.int64))
    return np.concatenate(keys) if keys else np.zeros(0, dtype=np.int64)


# -- bulk sampling -----------------------------------------------------------------


def sample_epoch_bulk(G: Graph, cfg: SamplerConfig, batches, epoch=0, batch_offset=0,
                      prob_spgemm=None, mode="auto") -> SampledEpoch:
    """Sample every layer for k minibatches in one stacked pass on the GPU
    (reference sampler.py:325-387).

    batch_offset: epoch-global index of batches[0] (keys line up across
    chunks).  prob_spgemm: the reference's hook to substitute the probability
    multiply; when given, P is materialised through it and normalised and
    sampled by the generic device kernels (ops.py), otherwise the fused
    device path runs.  mode (SAGE): "dedup" (default; Alg. 1 with every
    distinct P row formed on chip once), "stream" (Alg. 1, every P row
    streamed) or "pfree" (P-free exact fast path); LADIES: "race" / "exact"
    ("auto" picks exact replay on small graphs).  Outputs of the SAGE modes
    are identical.
    """
    from . import engine

    batches = [np.asarray(b, dtype=np.int64) for b in batches]
    if prob_spgemm is not None:
        return engine.sample_epoch_generic(G, cfg, batches, epoch, batch_offset, prob_spgemm)
    if cfg.kind is SamplerKind.SAGE:
        return engine.sage_epoch(G, cfg, batches, epoch, batch_offset,
                                 mode="dedup" if mode in ("auto", None) else mode)
    return engine.ladies_epoch(G, cfg, batches, epoch, batch_offset,
                               mode="auto" if mode in ("dedup", "stream", None) else mode)


# -- per-row samplers of the reference sampler.py, on the GPU (ops.py) ----------


def its_sample_row(probabilities, s, rng):
    from .ops import its_sample_row as _f

    return _f(probabilities, s, rng)


def sample_rows_ordered(P, s, epoch, layer, seed, row_keys=None):
    from .ops import sample_rows_ordered as _f

    return _f(P, s, epoch, layer, seed, row_keys)


def frontier_from_rows(sampled_rows, n_cols):
    from .ops import frontier_from_rows as _f

    return _f(sampled_rows, n_cols)


def sample_frontier(P, s, epoch, layer, seed, row_keys=None):
    from .ops import sample_frontier as _f

    return _f(P, s, epoch, layer, seed, row_keys)
