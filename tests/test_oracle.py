"""The oracle is pinned before it is trusted (task ③): the Philox restatement
against numpy's own Philox4x64-10 and the Random123 known answer, and the C
port of the sampler against golden outputs of the reference itself
(tests/golden/make_golden.py, reference run with injected uniforms)."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O
from oracle.philox import philox4x64_10, uniforms


def test_philox_random123_kat():
    out = philox4x64_10(np.zeros(4, np.uint64), np.zeros(2, np.uint64))
    assert [int(x) for x in out] == [
        0x16554D9ECA36314C, 0xDB20FE9D672D0FDC, 0xD7E772CEE186176B, 0x7E68B68AEC7BA23B]


def test_philox_matches_numpy_bitgenerator():
    rng = np.random.default_rng(0)
    for _ in range(100):
        ctr = rng.integers(0, 2**63, size=4, dtype=np.int64).astype(np.uint64)
        ctr[0] |= np.uint64(1)  # numpy pre-increments; avoid a borrow below
        key = rng.integers(0, 2**63, size=2, dtype=np.int64).astype(np.uint64)
        ref = np.random.Philox(key=key, counter=ctr - np.array([1, 0, 0, 0], np.uint64))
        assert np.array_equal(ref.random_raw(4), philox4x64_10(ctr, key))


def test_c_uniform_matches_numpy_restatement():
    rows = np.array([0, 1, 7, 2**40 + 3, 16_700_000_000])
    for t in range(9):
        want = uniforms(5, 2, 3, rows, t)
        got = [O.uniform(5, 2, 3, int(r), t) for r in rows]
        assert np.array_equal(want, np.array(got))


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "epoch_*.npz"))))
def test_oracle_matches_reference_golden(path):
    g, want = O.load_golden(path)
    if g["kind"] == "sage":
        got = O.sage_bulk(g["n"], g["rowptr"], g["col"], g["batches"], g["batch_size"],
                          g["fanouts"], g["seed"], g["epoch"], g["batch_offset"])
    else:
        got = O.ladies_bulk(g["n"], g["rowptr"], g["col"], g["batches"], g["fanouts"],
                            g["seed"], g["epoch"], g["batch_offset"])
    assert O.compare_epochs(want, got) == []


def test_oracle_its_matches_reference_rows():
    z = dict(np.load(os.path.join(GOLDEN, "its_rows.npz")))
    for i in range(len(z["deg"])):
        w = z["w_cat"][z["w_off"][i]:z["w_off"][i + 1]]
        want = z["picks"][i]
        want = want[want >= 0]
        assert np.array_equal(O.its_sample_row(w, int(z["fanout"][i]), z["u"][i]), want)


def test_oracle_threads_do_not_change_output():
    g, want = O.load_golden(os.path.join(GOLDEN, "epoch_rmat12_sage.npz"))
    for th in (1, 3):
        got = O.sage_bulk(g["n"], g["rowptr"], g["col"], g["batches"], g["batch_size"],
                          g["fanouts"], g["seed"], threads=th)
        assert O.compare_epochs(want, got) == []


def _pipeline_golden():
    z = dict(np.load(os.path.join(GOLDEN, "pipeline.npz")))
    return z


def _ragged(z, name):
    off, cat = z[name + "_off"], z[name + "_cat"]
    return [cat[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def test_pipeline_restatement_matches_reference_outputs():
    """oracle/pipeline_ref.py (the pipeline checker of the GPU tests) against
    the reference's own fetch_features + _propagate_batch outputs
    (pipeline.py:78-130, 273-305) on injected-uniform epochs, SAGE and
    LADIES — pins the pipeline oracle."""
    from oracle import pipeline_ref as PR

    z = _pipeline_golden()
    H = z["H"]
    for kind in ("sage", "ladies"):
        _, layers = O.load_golden(os.path.join(GOLDEN, "pipeline.npz"), prefix=f"{kind}_ep_")
        Y, Yoff = z[f"{kind}_Y"], z[f"{kind}_Yoff"]
        deep = layers[-1]
        for b in range(len(Yoff) - 1):
            X = H[deep["colv_cat"][deep["colv_off"][b]:deep["colv_off"][b + 1]]]
            got = PR.propagate_batch(layers, b, X)
            assert np.allclose(got, Y[Yoff[b]:Yoff[b + 1]], rtol=1e-12, atol=1e-12), (kind, b)


def test_pipeline_fetch_ledger_matches_reference():
    from oracle import pipeline_ref as PR

    z = _pipeline_golden()
    n = int(z["A_shape"][0])
    rs = np.linspace(0, n, 3).astype(np.int64)  # FeaturePartition bounds, 4 x 2 grid
    for req in range(4):
        want = PR.fetch_words(z["fetch_verts"], rs, z["H"].shape[1], 2, 2, req)
        for proc in range(4):
            m, w = want.get(proc, (0, 0))
            assert (m, w) == (z["fetch_msgs"][req, proc], z["fetch_words"][req, proc])
