"""ORACLE / TEST INFRASTRUCTURE ONLY.

numpy/scipy restatement of the reference epoch pipeline's data movement
(pkg/src/gnnbulk/pipeline.py), on the flat layer arrays of oracle.py
(LAYER_KEYS), float64 like the reference:

  * forward_aggregate      pipeline.py:123-130   A_l @ H_in
  * batch_block            pipeline.py:258-270   the batch's rows / columns
  * propagate_batch        pipeline.py:273-305   deepest layer first, carry by
                                                 first occurrence
  * fetch_words            pipeline.py:78-120 + dist.py:253-276  the
                           all-to-allv ledger charges of one fetch
  * trainer_of_batch       pipeline.py:184-197
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def forward_aggregate(n_rows, n_cols, ptr, col, H):
    """pipeline.py:123-130 (values 1.0)."""
    A = sp.csr_matrix((np.ones(len(col)), col, ptr), shape=(n_rows, n_cols))
    return np.asarray(A @ np.asarray(H, dtype=np.float64))


def batch_block(layer, b):
    """pipeline.py:258-270: rows r0:r1 of the stacked adjacency and the
    batch's column window (diagonal or shared layout)."""
    roff, coff = layer["rowv_off"], layer["colv_off"]
    r0, r1 = int(roff[b]), int(roff[b + 1])
    ncols_total = int(layer["adj_shape"][1])
    counts = np.diff(coff)
    if ncols_total == int(counts.sum()):
        c0, c1 = int(coff[b]), int(coff[b + 1])
    else:
        c0, c1 = 0, int(counts[b])
    ptr = layer["adj_ptr"][r0:r1 + 1]
    col = layer["adj_col"][ptr[0]:ptr[-1]]
    keep = (col >= c0) & (col < c1)
    # column_window keeps the window's entries, renumbered from c0
    rows = np.repeat(np.arange(r1 - r0), np.diff(ptr))
    kept_rows, kept_cols = rows[keep], col[keep] - c0
    nptr = np.zeros(r1 - r0 + 1, dtype=np.int64)
    np.add.at(nptr, kept_rows + 1, 1)
    return r1 - r0, c1 - c0, np.cumsum(nptr), kept_cols


def propagate_batch(layers, b, X):
    """pipeline.py:273-305 for batch b; X = rows of the deepest layer's
    col_vertices[b]."""
    Y = None
    for li in range(len(layers) - 1, -1, -1):
        layer = layers[li]
        R, C, ptr, col = batch_block(layer, b)
        Y = forward_aggregate(R, C, ptr, col, X)
        if li == 0:
            return Y
        deeper, shallower = layers[li], layers[li - 1]
        rows_of = deeper["rowv_cat"][deeper["rowv_off"][b]:deeper["rowv_off"][b + 1]]
        need = shallower["colv_cat"][shallower["colv_off"][b]:shallower["colv_off"][b + 1]]
        uniq, first = np.unique(rows_of, return_index=True)
        pos = np.searchsorted(uniq, need)
        X = Y[first[pos]]
    return Y


def fetch_words(vertices, row_starts, f, grid_rows, c, requester):
    """Ledger charges of fetch_features (sender -> (messages, words))."""
    vertices = np.asarray(vertices, dtype=np.int64)
    owner_rows = np.searchsorted(row_starts, vertices, side="right") - 1
    i_req, j_req = divmod(requester, c)
    out = {}
    for block_row in np.unique(owner_rows):
        owner = int(block_row) * c + j_req
        if owner == requester:
            continue
        out[owner] = (1, int(np.sum(owner_rows == block_row)) * f)
    return out


def trainer_of_batch(index_in_chunk, chunk_size, p, rows, c, replicated):
    """pipeline.py:184-197."""
    if replicated:
        bounds = np.linspace(0, chunk_size, p + 1).astype(np.int64)
        return int(np.searchsorted(bounds, index_in_chunk, side="right") - 1)
    row_bounds = np.linspace(0, chunk_size, rows + 1).astype(np.int64)
    row = int(np.searchsorted(row_bounds, index_in_chunk, side="right") - 1)
    within = index_in_chunk - int(row_bounds[row])
    row_count = int(row_bounds[row + 1] - row_bounds[row])
    rep_bounds = np.linspace(0, max(row_count, 1), c + 1).astype(np.int64)
    rep = int(np.searchsorted(rep_bounds, within, side="right") - 1)
    return row * c + rep
