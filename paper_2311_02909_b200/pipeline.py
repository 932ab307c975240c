"""End-to-end epoch driver (reference pkg/src/gnnbulk/pipeline.py): bulk
sampling, feature fetching, aggregation.

Same API and accounting as the reference; the data movement runs on the
device: feature rows are gathered from fp32 copies of the feature blocks in
HBM (`gb_gather_features`), and the aggregation chain of a whole bulk — every
minibatch at once over the stacked sampled adjacency — is `gb_spmm_rows`
plus the first-occurrence carry between layers (`gb_first_occurrence`).
Features are fp32 on the device (the reference computes in float64);
results agree within float32 rounding.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .errors import ContractViolation
from .sampler import SampledEpoch, SamplerConfig, SamplerKind, sample_epoch_bulk
from .sparse import SparseMatrix


def make_batches(train_vertices, batch_size: int, seed: int, epoch: int):
    """Deterministic shuffle of the training set into batches of b, the last
    possibly short (reference pipeline.py:171-181: numpy PCG64 keyed by
    SeedSequence([seed, 0x6261746368, epoch]))."""
    train = np.asarray(train_vertices, dtype=np.int64)
    order = np.random.Generator(
        np.random.PCG64(np.random.SeedSequence([seed, 0x6261746368, epoch]))
    ).permutation(len(train))
    shuffled = train[order]
    return [shuffled[i:i + batch_size] for i in range(0, len(shuffled), batch_size)]


# -- features (pipeline.py:33-120) -------------------------------------------------


@dataclass(frozen=True)
class FeaturePartition:
    """Dense n×f feature matrix split into grid.rows contiguous blocks; block
    i is replicated on the processes of grid row i (pipeline.py:33-75).  The
    device keeps one fp32 copy per block (`device_blocks`)."""

    grid: object
    blocks: tuple
    row_starts: np.ndarray
    _dev: list = field(default_factory=list, compare=False, repr=False)

    def __post_init__(self):
        if len(self.blocks) != self.grid.rows:
            raise ContractViolation("need one feature block per grid row")
        widths = {b.shape[1] for b in self.blocks}
        if len(widths) != 1 or widths.pop() < 1:
            raise ContractViolation("feature blocks must share a positive width")

    @classmethod
    def partition(cls, H, grid) -> "FeaturePartition":
        H = np.asarray(H, dtype=np.float64)
        if H.ndim != 2 or H.shape[1] < 1:
            raise ContractViolation("feature matrix must be n×f with f > 0")
        if H.shape[0] < grid.rows:
            raise ContractViolation("fewer feature rows than grid rows")
        bounds = np.linspace(0, H.shape[0], grid.rows + 1).astype(np.int64)
        blocks = tuple(H[bounds[i]:bounds[i + 1]].copy() for i in range(grid.rows))
        return cls(grid, blocks, bounds)

    @property
    def n(self) -> int:
        return int(self.row_starts[-1])

    @property
    def f(self) -> int:
        return self.blocks[0].shape[1]

    def owner_row(self, vertex: int) -> int:
        return int(np.searchsorted(self.row_starts, vertex, side="right") - 1)

    def full(self) -> np.ndarray:
        return np.concatenate(self.blocks, axis=0)

    def device_blocks64(self):
        """float64 copies of the blocks in HBM viewed as fp32 pairs (the
        reference's values, gathered bit for bit)."""
        import torch

        if not getattr(self, "_dev64", None):
            object.__setattr__(self, "_dev64", [
                torch.as_tensor(np.ascontiguousarray(b, dtype=np.float64)).cuda().view(
                    torch.float32) for b in self.blocks])
        return self._dev64

    def device_blocks(self):
        """fp32 copies of the blocks in HBM (built once)."""
        import torch

        if not self._dev:
            for b in self.blocks:
                self._dev.append(torch.as_tensor(np.ascontiguousarray(b, dtype=np.float32)).cuda())
        return self._dev


def _gather_rows(ids, H_dev, row0=0):
    """out[i] = H_dev[ids[i] - row0] on the device (gb_gather_features)."""
    import torch

    from . import _lib

    ids = torch.as_tensor(ids, dtype=torch.int32, device="cuda")
    f = H_dev.shape[1]
    out = torch.empty((ids.numel(), f), dtype=torch.float32, device="cuda")
    if ids.numel():
        _lib.check(_lib.lib().gb_gather_features(ids.numel(), _lib.ptr(ids), int(row0),
                                                 _lib.ptr(H_dev), f, _lib.ptr(out),
                                                 _lib.stream_ptr()))
    return out


def _charge_fetch(owner_rows, f, grid, ledger, requester):
    """The reference's all-to-allv word accounting for one fetch: every
    remote owner of the requester's grid column pays one message and
    (rows × f) words (pipeline.py:103-118, dist.py:253-276)."""
    if ledger is None or owner_rows.size == 0:
        return
    _, j_req = grid.coords(requester)
    rows, counts = np.unique(owner_rows, return_counts=True)
    for block_row, cnt in zip(rows, counts):
        owner = grid.rank(int(block_row), j_req)
        if owner != requester:
            ledger.charge(owner, "all-to-allv", 1, int(cnt) * f)


def fetch_features(frontier_vertices, Hpart: FeaturePartition, grid, ledger=None,
                   requester: int = 0) -> np.ndarray:
    """Feature rows of the given vertices onto one process, in the requested
    order, duplicates once per occurrence (pipeline.py:78-120).  Rows owned
    by the requester are free; the others are charged as the column
    all-to-allv.  Gathered on the device from the fp32 block copies."""
    import torch

    vertices = np.asarray(frontier_vertices, dtype=np.int64)
    if vertices.size and (vertices.min() < 0 or vertices.max() >= Hpart.n):
        raise ContractViolation("frontier vertex id out of range")
    owner_rows = (np.searchsorted(Hpart.row_starts, vertices, side="right") - 1
                  if vertices.size else np.zeros(0, dtype=np.int64))
    _charge_fetch(owner_rows, Hpart.f, grid, ledger, requester)
    # float64 rows gathered as raw bytes (two fp32 words each): exact
    out = torch.empty((vertices.size, 2 * Hpart.f), dtype=torch.float32, device="cuda")
    dev = Hpart.device_blocks64()
    for block_row in np.unique(owner_rows):
        sel = np.nonzero(owner_rows == block_row)[0]
        rows = _gather_rows(vertices[sel], dev[int(block_row)], Hpart.row_starts[block_row])
        out[torch.as_tensor(sel, device="cuda")] = rows
    return out.view(torch.float64).cpu().numpy()


def fetch_features_device(vertices, Hpart: FeaturePartition, grid, ledger=None, requester=0):
    """fetch_features with the rows left in HBM (fp32 tensor)."""
    import torch

    vertices = np.asarray(vertices, dtype=np.int64)
    owner_rows = (np.searchsorted(Hpart.row_starts, vertices, side="right") - 1
                  if vertices.size else np.zeros(0, dtype=np.int64))
    _charge_fetch(owner_rows, Hpart.f, grid, ledger, requester)
    out = torch.empty((vertices.size, Hpart.f), dtype=torch.float32, device="cuda")
    dev = Hpart.device_blocks()
    for block_row in np.unique(owner_rows):
        sel = np.nonzero(owner_rows == block_row)[0]
        rows = _gather_rows(vertices[sel], dev[int(block_row)], Hpart.row_starts[block_row])
        out[torch.as_tensor(sel, device="cuda")] = rows
    return out


# -- aggregation (pipeline.py:123-130, 258-305) ----------------------------------


def _spmm(R, rowptr, col, X, row_batch=None, shift=None, k=0):
    import torch

    from . import _lib

    f = X.shape[1]
    Y = torch.empty((R, f), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().gb_spmm_rows(
        R, _lib.ptr(rowptr), _lib.ptr(col), _lib.ptr(row_batch) if row_batch is not None else None,
        _lib.ptr(shift) if shift is not None else None, int(k), _lib.ptr(X), f, _lib.ptr(Y),
        _lib.stream_ptr()))
    return Y


def forward_aggregate(A_l: SparseMatrix, H_in) -> np.ndarray:
    """Aggregation product A_l @ H_in (sparse times dense), reference
    pipeline.py:123-130 — on the device in float64 with A's values, in
    scipy's accumulation order (gb_spmm_f64): bit-identical results."""
    import torch

    from . import _lib

    H_in = np.asarray(H_in, dtype=np.float64)
    if H_in.ndim != 2 or A_l.n_cols != H_in.shape[0]:
        raise ContractViolation(f"aggregation mismatch: {A_l.shape} @ {H_in.shape}")
    R, f = A_l.n_rows, H_in.shape[1]
    rowptr = torch.as_tensor(np.asarray(A_l.row_offsets, dtype=np.int64)).cuda()
    col = torch.as_tensor(np.asarray(A_l.col_indices, dtype=np.int32)).cuda() if A_l.nnz else \
        torch.zeros(1, dtype=torch.int32, device="cuda")
    val = torch.as_tensor(np.ascontiguousarray(A_l.values, dtype=np.float64)).cuda() if A_l.nnz \
        else torch.zeros(1, dtype=torch.float64, device="cuda")
    X = torch.as_tensor(np.ascontiguousarray(H_in)).cuda()
    Y = torch.empty((R, f), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().gb_spmm_f64(R, _lib.ptr(rowptr), _lib.ptr(col), _lib.ptr(val),
                                      _lib.ptr(X), f, _lib.ptr(Y), _lib.stream_ptr()),
               "gb_spmm_f64")
    return Y.cpu().numpy()


def _layer_shift(dev, k):
    """X row of a column index per batch: 0 for the block-diagonal layout,
    the batch's col-vertex offset for the shared one (_batch_block,
    pipeline.py:258-270)."""
    U = int(dev["colv_cat"].numel())
    if int(dev["adj_shape"][1]) == U:
        return None
    return dev["colv_off"][:k].contiguous()


def propagate_bulk(sampled: SampledEpoch, X):
    """The aggregation chain of every minibatch of a bulk at once (reference
    _propagate_batch, pipeline.py:273-305, applied to each batch): deepest
    layer first, Y = A^l X over the stacked adjacency, then each column
    vertex of the shallower layer takes the Y row of its first occurrence
    among the deeper layer's rows.  X: fp32 device rows of
    layers[-1].col_vertices stacked by batch.  Returns the layer-1 Y (device,
    rows = batch vertices stacked)."""
    import torch

    from . import _lib

    layers = sampled.layers
    if not all(_on_device(layer) for layer in layers):
        return _propagate_host_layers(sampled, X)
    k = len(sampled.batches)
    Y = None
    for li in range(len(layers) - 1, -1, -1):
        dev = layers[li].device
        R = int(dev["adj_shape"][0])
        if X.shape[0] != int(dev["colv_cat"].numel()):
            raise ContractViolation("feature rows must match the deepest col_vertices")
        Y = _spmm(R, dev["adj_ptr"], dev["adj_col"], X, dev["rowv_off"],
                  _layer_shift(dev, k), k)
        if li == 0:
            return Y
        sh = layers[li - 1].device
        U = int(sh["colv_cat"].numel())
        if sampled.kind is SamplerKind.LADIES:
            # the deeper rows are the shallower sampled sets, in order
            X = Y[:U]
            continue
        first = torch.empty(max(U, 1), dtype=torch.int32, device="cuda")
        F = int(sh["frontier_col"].numel())
        shift = _layer_shift(sh, k)
        _lib.check(_lib.lib().gb_first_occurrence(
            F, _lib.ptr(sh["adj_col"]), _lib.ptr(sh["sampv_off"]),
            _lib.ptr(shift) if shift is not None else None, k, U, _lib.ptr(first),
            _lib.stream_ptr()))
        X = _gather_rows(first[:U], Y)
    return Y


# -- epoch (pipeline.py:133-255) ---------------------------------------------------


@dataclass(frozen=True)
class EpochPlan:
    """Chunk schedule covering every training batch exactly once
    (pipeline.py:133-158)."""

    total_batches: int
    bulk_count: int
    chunks: tuple

    @classmethod
    def build(cls, total_batches: int, bulk_count: int) -> "EpochPlan":
        if total_batches < 0 or bulk_count < 1:
            raise ContractViolation("invalid epoch plan sizes")
        chunks = tuple((start, min(start + bulk_count, total_batches))
                       for start in range(0, total_batches, bulk_count))
        return cls(total_batches, bulk_count, chunks)

    @property
    def rounds(self) -> int:
        return len(self.chunks)


@dataclass
class EpochReport:
    """Outcome of one epoch (pipeline.py:160-169)."""

    epoch: int
    mode: str
    n_batches: int
    chunks: int
    spgemm_calls: int
    batches_per_process: list
    durations: dict
    ledger: object
    prediction: object = None


def _trainer_of_batch(index_in_chunk, chunk_size, grid, mode):
    """Deal a chunk's batches contiguously over trainers (pipeline.py:184-197)."""
    from .dist import MODE_REPLICATED

    if mode == MODE_REPLICATED:
        bounds = np.linspace(0, chunk_size, grid.p + 1).astype(np.int64)
        return int(np.searchsorted(bounds, index_in_chunk, side="right") - 1)
    row_bounds = np.linspace(0, chunk_size, grid.rows + 1).astype(np.int64)
    row = int(np.searchsorted(row_bounds, index_in_chunk, side="right") - 1)
    within = index_in_chunk - int(row_bounds[row])
    row_count = int(row_bounds[row + 1] - row_bounds[row])
    rep_bounds = np.linspace(0, max(row_count, 1), grid.c + 1).astype(np.int64)
    rep = int(np.searchsorted(rep_bounds, within, side="right") - 1)
    return grid.rank(row, rep)


def run_epoch(G, Hpart: FeaturePartition, cfg: SamplerConfig, grid, mode=None, epoch: int = 0,
              ledger=None, train_vertices=None, cost_params=None) -> EpochReport:
    """One epoch: chunked bulk sampling, then feature fetching and
    aggregation through every layer (pipeline.py:200-255).

    Each chunk's minibatches are fetched and propagated together on the
    device (one gather, one aggregation chain per chunk); batch-to-trainer
    assignment and the all-to-allv word charges are the reference's, per
    minibatch."""
    import torch

    from .dist import MODE_REPLICATED, CommLedger, predict_costs, sample_epoch_distributed

    mode = MODE_REPLICATED if mode is None else mode
    if train_vertices is None:
        train_vertices = np.arange(G.n)
    if ledger is None:
        ledger = CommLedger(grid.p)
    batches = make_batches(train_vertices, cfg.batch_size, cfg.seed, epoch)
    plan = EpochPlan.build(len(batches), cfg.bulk_count)
    durations = {"sample": 0.0, "fetch": 0.0, "propagate": 0.0}
    spgemm_calls = 0
    per_process = [0] * grid.p
    for start, stop in plan.chunks:
        chunk = batches[start:stop]
        t0 = time.perf_counter()
        if grid.p == 1:
            sampled = sample_epoch_bulk(G, cfg, chunk, epoch=epoch, batch_offset=start)
        else:
            sampled = sample_epoch_distributed(G, cfg, chunk, grid, mode=mode, epoch=epoch,
                                               batch_offset=start, ledger=ledger)
        torch.cuda.synchronize()
        durations["sample"] += time.perf_counter() - t0
        spgemm_calls += sampled.spgemm_calls
        t0 = time.perf_counter()
        deepest = sampled.layers[-1]
        a = deepest.to_arrays()
        cat, off = a["colv_cat"], a["colv_off"]
        owner_rows = np.searchsorted(Hpart.row_starts, cat, side="right") - 1
        for local in range(len(chunk)):
            trainer = _trainer_of_batch(local, len(chunk), grid, mode)
            per_process[trainer] += 1
            _charge_fetch(owner_rows[off[local]:off[local + 1]], Hpart.f, grid, ledger, trainer)
        X = fetch_features_device(cat, Hpart, grid, None, 0)
        torch.cuda.synchronize()
        durations["fetch"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        if all(_on_device(layer) for layer in sampled.layers):
            propagate_bulk(sampled, X)
        else:
            _propagate_host_layers(sampled, X)
        torch.cuda.synchronize()
        durations["propagate"] += time.perf_counter() - t0
    prediction = predict_costs(cost_params) if cost_params is not None else None
    return EpochReport(epoch=epoch, mode=mode, n_batches=len(batches), chunks=plan.rounds,
                       spgemm_calls=spgemm_calls, batches_per_process=per_process,
                       durations=durations, ledger=ledger, prediction=prediction)


def _on_device(layer):
    import torch

    return layer.device is not None and isinstance(layer.device.get("adj_col"), torch.Tensor)


def _propagate_host_layers(sampled: SampledEpoch, X):
    """Results assembled on the host (the distributed simulator): upload the
    layers, then the same device chain."""
    import torch

    from .sampler import LayerSample

    layers = []
    for layer in sampled.layers:
        a = layer.to_arrays()
        dev = {}
        for key, v in a.items():
            if key.endswith("_shape"):
                dev[key] = tuple(int(x) for x in v)
            elif key.endswith(("_ptr", "_off")):
                dev[key] = torch.as_tensor(v.astype(np.int64)).cuda()
            else:
                dev[key] = torch.as_tensor(v.astype(np.int32)).cuda() if v.size else \
                    torch.zeros(1, dtype=torch.int32, device="cuda")[:0]
        layers.append(LayerSample(layer.depth, device=dev))
    return propagate_bulk(SampledEpoch(sampled.kind, sampled.epoch, sampled.batches, layers,
                                       len(layers)), X)
