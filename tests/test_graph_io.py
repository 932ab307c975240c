"""Host side of graph ingestion and the drop-in name surface (CPU): file
tokenising and its GraphFormatError texts (reference pkg/tests/test_io.py),
RunConfig validation, stats records, the oracle's synthetic-graph recipe,
and that the package exports every public name of the reference
(`pkg/src/gnnbulk/__init__.py:11-79`)."""

import numpy as np
import pytest

import paper_2311_02909_b200 as gb
from paper_2311_02909_b200 import graph_io as gio

# reference pkg/src/gnnbulk/__init__.py:11-77 (public names)
REFERENCE_NAMES = """ContractViolation GraphFormatError Graph SparseMatrix add block_diag
build_column_extraction column_window compact_columns expand_row_extraction norm_rows_ladies
norm_rows_sage rows_subset spgemm vstack LayerSample RowRng SampledEpoch SamplerConfig
SamplerKind frontier_from_rows its_sample_row ladies_seed_matrix sage_seed_matrix
sample_epoch_bulk sample_frontier sample_rows_ordered MODE_PARTITIONED MODE_REPLICATED PHASES
CommLedger CostModelParams CostPrediction Mailbox Partition1_5D ProcessGrid StageTransfer
allreduce_sum alltoallv partition_block_rows partition_from_blocks predict_costs
replicated_spgemm sample_epoch_distributed spgemm_15d_sparsity_aware EpochPlan EpochReport
FeaturePartition fetch_features forward_aggregate make_batches run_epoch RunConfig emit_stats
load_graph read_stats save_graph synthesize_features""".split()


def test_top_level_names_match_reference():
    missing = [n for n in REFERENCE_NAMES if not hasattr(gb, n)]
    assert missing == []


FIGURE = [(0, 1), (1, 0), (1, 4), (4, 1), (2, 5), (5, 2), (3, 5), (5, 3), (4, 5), (5, 4)]


def _write(path, lines):
    path.write_text("\n".join(lines) + "\n")


def test_edge_list_tokens(tmp_path):
    p = tmp_path / "g.txt"
    _write(p, ["# demo", "# n=8"] + [f"{u} {v}" for u, v in FIGURE] + ["", "   "])
    n, s, d = gio._edge_list(p)
    assert n == 8 and s.tolist() == [u for u, _ in FIGURE] and d.tolist() == [v for _, v in FIGURE]
    _write(p, [f"{u} {v}" for u, v in FIGURE])
    assert gio._edge_list(p)[0] == 6


@pytest.mark.parametrize("lines,where", [
    (["0 1", "1 2 3"], ":2:"),
    (["0 x"], ":1:"),
    (["0 1", "-1 2"], ":2:"),
    (["# n=abc", "0 1"], ":1:"),
])
def test_edge_list_errors_carry_line(tmp_path, lines, where):
    p = tmp_path / "bad.txt"
    _write(p, lines)
    with pytest.raises(gb.GraphFormatError, match=where):
        gio._edge_list(p)


def test_edge_list_header_and_empty(tmp_path):
    p = tmp_path / "h.txt"
    _write(p, ["# n=2", "0 5"])
    with pytest.raises(gb.GraphFormatError, match="exceeds declared n=2"):
        gio._edge_list(p)
    _write(p, ["# nothing"])
    with pytest.raises(gb.GraphFormatError, match="empty edge list"):
        gio._edge_list(p)
    _write(p, ["# n=4"])
    n, s, d = gio._edge_list(p)
    assert n == 4 and s.size == 0


def test_matrix_market_tokens_and_errors(tmp_path):
    p = tmp_path / "g.mtx"
    _write(p, ["%%MatrixMarket matrix coordinate pattern symmetric", "% c", "3 3 2", "2 1", "3 3"])
    n, s, d = gio._matrix_market(p)
    assert n == 3 and sorted(zip(s.tolist(), d.tolist())) == [(0, 1), (1, 0), (2, 2)]
    _write(p, ["%%MatrixMarket matrix coordinate real general", "2 2 1", "1 2 0.5"])
    assert gio._matrix_market(p)[0] == 2
    for lines, msg in ((["%%MatrixMarket matrix array real general"], ":1:"),
                       (["not a banner"], "banner"),
                       (["%%MatrixMarket matrix coordinate pattern general", "2 3 1"], "square"),
                       (["%%MatrixMarket matrix coordinate pattern general", "2 2 1", "3 1"],
                        "out of range"),
                       (["%%MatrixMarket matrix coordinate pattern general"], "missing size")):
        _write(p, lines)
        with pytest.raises(gb.GraphFormatError, match=msg):
            gio._matrix_market(p)


def test_load_graph_rejects_unknown_format(tmp_path):
    with pytest.raises(gb.ContractViolation):
        gb.load_graph(tmp_path / "x", fmt="csv")
    with pytest.raises(gb.ContractViolation):
        gb.load_graph(tmp_path / "x", direction="both")


def test_run_config_rules():
    cfg = gb.RunConfig("g.txt", layers=3, sample_num=4)
    assert cfg.fanouts == (4, 4, 4) and cfg.as_dict()["fanouts"] == [4, 4, 4]
    for kw in ({"format": "csv"}, {"sampler": "gat"}, {"mode": "x"}, {"direction": "up"},
               {"layers": 0}, {"fanouts": (1, 2), "layers": 3}, {"procs": 3, "replication": 2}):
        with pytest.raises(gb.ContractViolation):
            gb.RunConfig("g.txt", **kw)


def test_synthesize_features_matches_reference_stream():
    x = gb.synthesize_features(5, 3, 7)
    g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([7, 0x66656174])))
    assert np.array_equal(x, g.standard_normal((5, 3)))
    with pytest.raises(gb.ContractViolation):
        gb.synthesize_features(0, 3, 1)


def test_stats_round_trip(tmp_path):
    from paper_2311_02909_b200.pipeline import EpochReport

    led = gb.CommLedger(2)
    led.charge(1, "row-data", 2, 40)
    rep = EpochReport(0, "replicated", 4, 2, 6, [2, 2], {"sample": 0.5}, led)
    path = tmp_path / "s.jsonl"
    gb.emit_stats(rep, path, gb.RunConfig("g.txt"))
    recs = gb.read_stats(path)
    assert [r["record"] for r in recs] == ["run", "epoch"] + ["phase"] * 8
    ep = recs[1]
    assert tuple(ep) == gio.STATS_EPOCH_FIELDS
    assert ep["words"]["row-data"] == 40 and ep["predicted"] is None
    assert tuple(recs[2]) == gio.STATS_PHASE_FIELDS


def test_oracle_generator_is_a_canonical_graph():
    from oracle import oracle as O

    n, m = 4096, 30000
    rowptr, col = O.rmat_graph(n, m, symmetric=True, seed=3)
    assert rowptr[-1] == 2 * m and rowptr[0] == 0
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    assert np.all((rows[1:] > rows[:-1]) | (col[1:] > col[:-1]))  # sorted, distinct
    assert not np.any(rows == col)
    fwd = set(zip(rows.tolist(), col.tolist()))
    assert all((v, u) in fwd for u, v in list(fwd)[:2000])
    r2, c2 = O.rmat_graph(n, m, symmetric=False, seed=3)
    assert r2[-1] == m
