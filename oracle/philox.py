"""ORACLE / TEST INFRASTRUCTURE ONLY — never imported by the product path.

Vectorised numpy restatement of the counter-based uniform source that both
the CUDA sampler and the injected CPU oracle consume.

Why it exists: the reference keys one PCG64 stream per
(seed, epoch, layer, global_row) (`pkg/src/gnnbulk/sampler.py:97-116`,
`RowRng.stream`).  Its stream values are not pinned by any golden vector
(SURVEY.md §8(c)), so bit-exact parity is done by *injecting* one shared
counter-based function into both sides:

    u(seed, epoch, depth, row, t) =
        (Philox4x64-10(ctr=[row, depth, t >> 2, 0], key=[seed, epoch])[t & 3] >> 11) * 2**-53

Philox4x64-10 is the Random123 generator that numpy ships as
`numpy.random.Philox` (third-party, numpy 2.3.5 here).  This file is pinned
against `numpy.random.Philox` itself in `tests/test_oracle.py` (numpy
pre-increments its counter, so numpy's counter c yields our block c+1) and
against the Random123 known-answer vector (ctr=0, key=0).
"""

from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2E7470EE14C6C93)
M1 = np.uint64(0xCA5A826395121157)
W0 = np.uint64(0x9E3779B97F4A7C15)
W1 = np.uint64(0xBB67AE8584CAA73B)
_MASK32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def _mulhilo64(a: np.uint64, b: np.ndarray):
    """128-bit product of uint64 scalar a and uint64 array b -> (hi, lo)."""
    b = b.astype(np.uint64)
    a_lo, a_hi = a & _MASK32, a >> _S32
    b_lo, b_hi = b & _MASK32, b >> _S32
    with np.errstate(over="ignore"):
        ll = a_lo * b_lo
        lh = a_lo * b_hi
        hl = a_hi * b_lo
        hh = a_hi * b_hi
        mid = (ll >> _S32) + (lh & _MASK32) + (hl & _MASK32)
        hi = hh + (lh >> _S32) + (hl >> _S32) + (mid >> _S32)
        lo = a * b
    return hi, lo


def philox4x64_10(ctr, key):
    """Raw Philox4x64 with 10 rounds.

    ctr: uint64 array (..., 4); key: uint64 array (..., 2) (broadcastable).
    Returns uint64 array (..., 4).  No counter pre-increment.
    """
    ctr = np.asarray(ctr, dtype=np.uint64)
    key = np.asarray(key, dtype=np.uint64)
    shape = np.broadcast_shapes(ctr.shape[:-1], key.shape[:-1])
    c0, c1, c2, c3 = (np.broadcast_to(ctr[..., i], shape).copy() for i in range(4))
    k0 = np.broadcast_to(key[..., 0], shape).copy()
    k1 = np.broadcast_to(key[..., 1], shape).copy()
    with np.errstate(over="ignore"):
        for r in range(10):
            if r:
                k0 = k0 + W0
                k1 = k1 + W1
            hi0, lo0 = _mulhilo64(M0, c0)
            hi1, lo1 = _mulhilo64(M1, c2)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return np.stack([c0, c1, c2, c3], axis=-1)


def uniforms(seed, epoch, depth, rows, t):
    """u(seed, epoch, depth, row, t) for broadcastable integer arrays rows, t.

    Returns float64 values in [0, 1) with 53 random bits.
    """
    rows = np.asarray(rows, dtype=np.int64).astype(np.uint64)
    t = np.asarray(t, dtype=np.int64)
    rows, t = np.broadcast_arrays(rows, t)
    ctr = np.stack(
        [
            rows,
            np.full(rows.shape, np.uint64(int(depth) & 0xFFFFFFFFFFFFFFFF)),
            (t >> 2).astype(np.uint64),
            np.zeros(rows.shape, dtype=np.uint64),
        ],
        axis=-1,
    )
    key = np.array([int(seed) & 0xFFFFFFFFFFFFFFFF, int(epoch) & 0xFFFFFFFFFFFFFFFF],
                   dtype=np.uint64)
    out = philox4x64_10(ctr, key)
    word = np.take_along_axis(out, (t & 3)[..., None].astype(np.int64), axis=-1)[..., 0]
    return (word >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


class InjectedStream:
    """Drop-in for the numpy Generator returned by reference `RowRng.stream`
    (`sampler.py:112-116`): successive `.random()` calls return
    u(seed, epoch, layer, row, 0), u(..., 1), ...  (the t-th draw of the row,
    exactly as `its_sample_row` consumes them, `sampler.py:176-181`)."""

    __slots__ = ("seed", "epoch", "layer", "row", "t")

    def __init__(self, seed, epoch, layer, row):
        self.seed, self.epoch, self.layer, self.row = seed, epoch, layer, int(row)
        self.t = 0

    def random(self, size=None):
        if size is None:
            u = float(uniforms(self.seed, self.epoch, self.layer, self.row, self.t))
            self.t += 1
            return u
        size = int(size)
        ts = np.arange(self.t, self.t + size)
        self.t += size
        return uniforms(self.seed, self.epoch, self.layer, self.row, ts)
