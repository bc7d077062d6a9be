"""join_aggregate_both (P/src/engine.cpp:537-722).

CPU: the Python restatement (oracle/oracle.py oracle_aggregate) is pinned
against the reference library itself, bit for bit, on the reference test's
own instances (P/tests/test_engine.cpp:309-348: seed 508, values
unit()*10-5) for every (combine, agg) pair. GPU: the CUDA path equals the
reference's doubles exactly (same accumulation order, no FMA), plus the
report fields, the dense/sparse split, the classical rejection
(test_engine.cpp:350-359) and the CLI's hand-checkable rows
(test_cli.cpp:217-229)."""
import numpy as np
import pytest

import paper_2206_04995_b200 as d3
from oracle import oracle as O
from support import SplitMix64, random_instance

C = d3.CostConstants.test_consts()
AGGS = ["sum", "count", "min", "max", "avg"]
COMBINES = ["multiply", "add", "abs_diff", "left", "right"]


def attach_values(n, rng):
    """attach_values (test_engine.cpp:34-40): unit() * 10 - 5 per row."""
    return np.array([rng.unit() * 10.0 - 5.0 for _ in range(n)], dtype=np.float64)


def _instances(seed, count, max_card=48, max_rows=600):
    rng = SplitMix64(seed)
    out = []
    for _ in range(count):
        r, s = random_instance(rng, max_card, max_rows)
        rv = attach_values(len(r[0]), rng)
        sv = attach_values(len(s[0]), rng)
        out.append((r, s, rv, sv))
    return out


def _same(a: dict, b: dict):
    assert a.keys() == b.keys()
    for k in a:
        x, y = a[k], b[k]
        assert (x == y) or (x != x and y != y), (k, x, y)  # bit-equal or both NaN
        assert np.float64(x).tobytes() == np.float64(y).tobytes() or x != x, (k, x, y)


# ---- CPU: pin the restatement against the reference ---------------------------
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_restatement_matches_reference_library():
    for r, s, rv, sv in _instances(508, 4):
        R, S = O.Table(*r), O.Table(*s)
        for cf in COMBINES:
            for af in AGGS:
                ref = O.ref_join_aggregate(R, S, rv, sv, cf, af)
                assert ref["strategy"] in (b"hybrid", "hybrid")
                _same(O.oracle_aggregate(R, S, rv, sv, cf, af), ref["cells"])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_rejects_classical_force():
    (r, s, rv, sv), = _instances(509, 1, 32, 200)
    with pytest.raises(O.ConfigErrorLike):
        O.ref_join_aggregate(O.Table(*r), O.Table(*s), rv, sv, "add", "sum", force="classical")


def test_python_mirror_validates_before_device_work():
    t = d3.RawTable(np.array([1, 2], np.uint64), np.array([3, 4], np.uint64))
    with pytest.raises(d3.ConfigError):
        d3.ValuedTable(t, np.array([1.0]))
    v = d3.ValuedTable(t, np.array([1.0, 2.0]))
    with pytest.raises(d3.ConfigError):
        d3.join_aggregate_both(v, v, d3.CombineFn.add, d3.AggFn.sum,
                               d3.EngineConfig(force=d3.Strategy.classical), C)
    assert d3.agg_from_name("avg") == d3.AggFn.avg and d3.agg_from_name("median") is None
    assert d3.combine_from_name("abs_diff") == d3.CombineFn.abs_diff


# ---- GPU ---------------------------------------------------------------------
def _gpu(r, s, rv, sv, cf, af, **kw):
    cfg = d3.EngineConfig(**kw)
    out = d3.join_aggregate_both(d3.ValuedTable(d3.RawTable(*r), rv),
                                 d3.ValuedTable(d3.RawTable(*s), sv),
                                 d3.CombineFn[cf], d3.AggFn[af], cfg, C)
    raw = d3.aggregate_to_raw(out)
    cells = {(int(a), int(b)): float(v) for a, b, v in zip(raw.raw_x, raw.raw_z, out.values)}
    assert len(cells) == raw.count == out.report.out_p
    return cells, out.report


@pytest.mark.gpu
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_every_function_pair_matches_reference_bitwise():
    """test_engine.cpp:309-348, exact doubles instead of Approx."""
    for r, s, rv, sv in _instances(508, 4):
        R, S = O.Table(*r), O.Table(*s)
        for cf in COMBINES:
            for af in AGGS:
                ref = O.ref_join_aggregate(R, S, rv, sv, cf, af)
                got, rep = _gpu(r, s, rv, sv, cf, af)
                _same(got, ref["cells"])
                assert rep.strategy == "hybrid"
                for k in ("out_p", "pairs_sparse", "pairs_dense", "dense_z", "sparse_z",
                          "f2_evaluations", "dropped_r", "x_card", "y_card", "z_card",
                          "out_j_estimate"):
                    assert getattr(rep, k) == ref[k], k


@pytest.mark.gpu
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("force", ["hybrid", "sparse", "dense"])
def test_forced_partitions_and_larger_instances(force):
    """Every force on larger random instances (duplicates, dictionary and
    natural keys, dropped R rows): values and the dense/sparse split equal
    the reference's."""
    fmap = {"hybrid": d3.Strategy.hybrid, "sparse": d3.Strategy.sparse_only,
            "dense": d3.Strategy.dense_only}
    for r, s, rv, sv in _instances(511, 6, 256, 5000):
        R, S = O.Table(*r), O.Table(*s)
        for cf, af in (("multiply", "sum"), ("add", "avg"), ("abs_diff", "max"),
                       ("right", "min"), ("left", "count")):
            ref = O.ref_join_aggregate(R, S, rv, sv, cf, af, force=force)
            got, rep = _gpu(r, s, rv, sv, cf, af, force=fmap[force])
            _same(got, ref["cells"])
            assert (rep.pairs_sparse, rep.pairs_dense, rep.dense_z) == \
                (ref["pairs_sparse"], ref["pairs_dense"], ref["dense_z"])


@pytest.mark.gpu
def test_special_values_and_count_only():
    """NaN, infinities and signed zeros go through combine/min/max exactly as
    std::min/std::max/IEEE do; count_only returns the same count."""
    r = (np.array([1, 1, 2, 2, 3], np.uint64), np.array([10, 10, 10, 11, 11], np.uint64))
    s = (np.array([5, 5, 6, 7], np.uint64), np.array([10, 10, 11, 11], np.uint64))
    rv = np.array([np.nan, -0.0, np.inf, 2.5, -np.inf])
    sv = np.array([0.0, -1.5, np.nan, 3.0])
    for cf in COMBINES:
        for af in AGGS:
            want = O.oracle_aggregate(O.Table(*r), O.Table(*s), rv, sv, cf, af)
            got, rep = _gpu(r, s, rv, sv, cf, af)
            _same(got, want)
            cnt = d3.join_aggregate_both(d3.ValuedTable(d3.RawTable(*r), rv),
                                         d3.ValuedTable(d3.RawTable(*s), sv), d3.CombineFn[cf],
                                         d3.AggFn[af], d3.EngineConfig(count_only=True), C)
            assert cnt.report.out_p == len(want) and not cnt.base.materialized


@pytest.mark.gpu
def test_cli_hand_checkable_rows(tmp_path):
    """test_cli.cpp:217-229: R = {(1,10,2),(2,10,4)}, S = {(5,10,3)}, avg of
    multiply -> rows "1\\t5\\t6", "2\\t5\\t12"."""
    r = d3.ValuedTable(d3.RawTable(np.array([1, 2], np.uint64), np.array([10, 10], np.uint64)),
                       np.array([2.0, 4.0]))
    s = d3.ValuedTable(d3.RawTable(np.array([5], np.uint64), np.array([10], np.uint64)),
                       np.array([3.0]))
    out = d3.join_aggregate_both(r, s, d3.CombineFn.multiply, d3.AggFn.avg, d3.EngineConfig(), C)
    assert out.report.out_p == 2
    rows = sorted(zip(out.base.raw_x.tolist(), out.base.raw_z.tolist(), out.values.tolist()))
    assert rows == [(1, 5, 6.0), (2, 5, 12.0)]


@pytest.mark.gpu
def test_device_resident_valued_tables():
    import torch
    (r, s, rv, sv), = _instances(512, 1)
    host, _ = _gpu(r, s, rv, sv, "multiply", "sum")
    dev = torch.device("cuda", 0)
    R = d3.ValuedTable(d3.RawTable(torch.tensor(r[0].view(np.int64), device=dev),
                                   torch.tensor(r[1].view(np.int64), device=dev)),
                       torch.tensor(rv, device=dev))
    S = d3.ValuedTable(d3.RawTable(torch.tensor(s[0].view(np.int64), device=dev),
                                   torch.tensor(s[1].view(np.int64), device=dev)),
                       torch.tensor(sv, device=dev))
    out = d3.join_aggregate_both(R, S, d3.CombineFn.multiply, d3.AggFn.sum, d3.EngineConfig(), C)
    got = {(int(a), int(b)): float(v) for a, b, v in zip(out.base.raw_x, out.base.raw_z, out.values)}
    _same(got, host)
