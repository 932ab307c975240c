"""Host-side process-grid logic (reference pkg/tests/test_dist.py
TestProcessGrid / TestPartition / collectives / cost model) — CPU only."""

import math

import numpy as np
import pytest

import paper_2311_02909_b200 as gb
from paper_2311_02909_b200.dist import (
    CommLedger,
    CostModelParams,
    Mailbox,
    ProcessGrid,
    alltoallv,
    partition_block_rows,
    predict_costs,
)


def test_grid_layout_round_trip():
    grid = ProcessGrid(8, 2)
    assert grid.rows == 4 and grid.stages == 2
    for r in range(8):
        assert grid.rank(*grid.coords(r)) == r
    assert grid.row_group(1) == [2, 3]
    assert grid.col_group(1) == [1, 3, 5, 7]


def test_grid_invariants():
    for p, c in ((6, 4), (4, 4), (0, 1), (2, 2)):
        with pytest.raises(gb.ContractViolation):
            ProcessGrid(p, c)
    assert ProcessGrid(4, 1).stages == 4 and ProcessGrid(1, 1).stages == 1


def test_partition_even_and_reconstruct():
    rng = np.random.default_rng(0)
    for rows, p, c in ((9, 4, 2), (17, 8, 2), (8, 4, 1)):
        dense = np.where(rng.random((rows, 7)) < 0.4, 1.0, 0.0)
        m = gb.SparseMatrix.from_dense(dense)
        part = partition_block_rows(m, ProcessGrid(p, c))
        heights = [b.n_rows for b in part.blocks]
        assert max(heights) - min(heights) <= 1 and sum(heights) == rows
        assert part.owner_row(0) == 0 and part.owner_row(rows - 1) == len(heights) - 1
    with pytest.raises(gb.ContractViolation):
        partition_block_rows(gb.SparseMatrix.identity(2), ProcessGrid(4, 1))


def test_mailbox_orders_by_sender():
    box = Mailbox()
    box.post(3, 0, "t", "c")
    box.post(1, 0, "t", "a")
    box.post(2, 0, "t", "b")
    assert [p for _, p in box.collect(0, "t")] == ["a", "b", "c"]
    assert box.collect(0, "t") == []


def test_alltoallv_charges_remote_words_only():
    led = CommLedger(4)
    out = alltoallv({0: {0: np.ones(3), 1: np.ones(2)}, 1: {0: np.ones(5)}}, [0, 1], led)
    assert [s for s, _ in out[0]] == [0, 1]
    assert led.words("all-to-allv", 0) == 2 and led.words("all-to-allv", 1) == 5
    assert led.messages() == 2
    with pytest.raises(gb.ContractViolation):
        alltoallv({5: {0: np.ones(1)}}, [0, 1])


def test_ledger_and_cost_model():
    led = CommLedger(2, alpha=2.0, beta=0.5)
    led.charge(0, "row-data", 2, 10)
    assert led.cost(0) == 2 * 2.0 + 10 * 0.5
    with pytest.raises(gb.ContractViolation):
        led.charge(0, "bogus", 1, 1)
    # the reference's worked example (pkg/tests/test_dist.py:292-296)
    pred = predict_costs(CostModelParams(p=4, c=1, k=1, b=2, s=2, d=3.0))
    assert pred.t_prob == pytest.approx(11.5)
    assert pred.t_rowdata == pytest.approx(math.log2(4) + 6.0)
    assert pred.t_allreduce == pytest.approx(1.5)
    pred = predict_costs(CostModelParams(p=8, c=2, k=4, b=2, s=1, d=1.5))
    kbd = 4 * 2 * 1.5
    assert pred.t_prob == pytest.approx(2 + math.log2(2) + kbd / 2 + 2 * kbd / 8)
    with pytest.raises(gb.ContractViolation):
        CostModelParams(p=2, c=2, k=1, b=1, s=1, d=1.0)
