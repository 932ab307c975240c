"""Epoch driver pieces that feed the sampler (reference pkg/src/gnnbulk/pipeline.py)."""

from __future__ import annotations

import numpy as np


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
