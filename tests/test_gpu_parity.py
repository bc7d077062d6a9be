"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
the reference's own randomized corpora and known-answer instances."""
import numpy as np
import pytest

import paper_2206_04995_b200 as d3
from oracle import oracle as O
from support import SplitMix64, oracle_pairs, pair_set, random_instance

pytestmark = pytest.mark.gpu
C = d3.CostConstants.test_consts()
FORCES = [d3.Strategy.hybrid, d3.Strategy.sparse_only, d3.Strategy.dense_only, d3.Strategy.classical,
          d3.Strategy.auto_select]


def _run(r, s, force, count_only=False, checksum=False, **kw):
    cfg = d3.EngineConfig(force=force, count_only=count_only, checksum=checksum, **kw)
    return d3.join_project(d3.RawTable(*r), d3.RawTable(*s), cfg, C)


@pytest.mark.parametrize("seed", [41, 501, 502])
def test_corpus_matches_oracle(seed):
    """acceptance criterion 1 / test_engine.cpp:89-113: every strategy equals
    the brute-force oracle."""
    rng = SplitMix64(seed)
    for _ in range(25):
        r, s = random_instance(rng)
        want = oracle_pairs(r, s)
        for f in FORCES:
            out = _run(r, s, f)
            assert out.report.out_p == len(want)
            assert pair_set(out.result.raw_x, out.result.raw_z) == want


def test_partition_and_stats_match_oracle():
    rng = SplitMix64(201)
    for _ in range(20):
        r, s = random_instance(rng, 128, 2000)
        o = O.orc_join_project(O.Table(*r), O.Table(*s), force="hybrid")
        g = _run(r, s, d3.Strategy.hybrid, count_only=True, checksum=True).report
        for k in ("x_card", "y_card", "z_card", "r_nnz", "s_nnz", "out_j", "dense_z",
                  "sparse_z", "pairs_sparse", "pairs_dense", "dropped_r", "spa_inner_count",
                  "f2_evaluations", "out_j_estimate", "checksum_sum", "checksum_xor",
                  "panel_bytes", "x_live"):
            assert g.__dict__[k] == o[k], k
        assert g.f1_value == o["f1"]


def test_cfg1_golden():
    """cfg1: count 9,429,141, sum 0x6f2f5d2033c05da4, xor 0x50caa74071957968."""
    r, s = O.gen(1, 0), O.gen(1, 1)
    out = _run((r.left, r.right), (s.left, s.right), d3.Strategy.hybrid, count_only=True,
               checksum=True)
    assert out.report.out_p == 9429141
    assert out.report.checksum_sum == 0x6F2F5D2033C05DA4
    assert out.report.checksum_xor == 0x50CAA74071957968
    assert out.report.dense_z == 9888 and out.report.sparse_z == 112
    full = _run((r.left, r.right), (s.left, s.right), d3.Strategy.hybrid)
    assert full.result.count == 9429141
    n, x, sm = O.set_fingerprint(full.result.raw_x, full.result.raw_z)
    assert (n, x, sm) == (9429141, 0x50CAA74071957968, 0x6F2F5D2033C05DA4)


def test_spec_known_answer():
    """SPEC.md:358 instance: R={(0,0),(0,1),(1,1)}, S rows y0->z0, y1->z0, y1->z1."""
    r = (np.array([0, 0, 1], np.uint64), np.array([0, 1, 1], np.uint64))
    s = (np.array([0, 0, 1], np.uint64), np.array([0, 1, 1], np.uint64))
    for f in FORCES:
        out = _run(r, s, f)
        assert pair_set(out.result.raw_x, out.result.raw_z) == {(0, 0), (0, 1), (1, 0), (1, 1)}


def test_cli_fixture_count():
    """test_cli.cpp:67-84: R={(1,10),(1,11),(2,10)}, S={(5,10),(6,11),(6,10)} -> 4."""
    r = (np.array([1, 1, 2], np.uint64), np.array([10, 11, 10], np.uint64))
    s = (np.array([5, 6, 6], np.uint64), np.array([10, 11, 10], np.uint64))
    assert _run(r, s, d3.Strategy.auto_select, count_only=True).report.out_p == 4


def test_empty_and_swap():
    e = (np.zeros(0, np.uint64), np.zeros(0, np.uint64))
    r = (np.array([1, 2], np.uint64), np.array([10, 11], np.uint64))
    assert _run(e, e, d3.Strategy.hybrid).report.out_p == 0
    assert _run(r, e, d3.Strategy.hybrid).report.out_p == 0
    big = (np.arange(100, 200, dtype=np.uint64), (10 + np.arange(100) % 2).astype(np.uint64))
    out = _run(r, big, d3.Strategy.hybrid)
    assert out.report.swapped
    assert pair_set(out.result.raw_x, out.result.raw_z) == oracle_pairs(r, big)


def test_natural_key_fallback_and_errors():
    i = np.arange(400, dtype=np.uint64)
    r = (i % 37, i % 23)
    s = (i % 31, i % 23)
    want = oracle_pairs(r, s)
    out = _run(r, s, d3.Strategy.hybrid)
    assert pair_set(out.result.raw_x, out.result.raw_z) == want
    cfg = d3.EngineConfig(force=d3.Strategy.hybrid, natural_keys_declared=d3.SkipFlags(True, True, True))
    out = d3.join_project(d3.RawTable(*r), d3.RawTable(*s), cfg, C)
    assert pair_set(out.result.raw_x, out.result.raw_z) == want
    huge = (r[0].copy(), r[1])
    huge[0][0] = 1 << 33
    with pytest.raises(d3.ConfigError):
        d3.join_project(d3.RawTable(*huge), d3.RawTable(*s), cfg, C)
    # auto-detected skip that fails the full scan falls back to dictionaries
    auto = d3.join_project(d3.RawTable(*huge), d3.RawTable(*s), d3.EngineConfig(force=d3.Strategy.hybrid), C)
    assert pair_set(auto.result.raw_x, auto.result.raw_z) == oracle_pairs(huge, s)
    with pytest.raises(d3.ConfigError):
        d3.join_project(d3.RawTable(*r), d3.RawTable(*s), d3.EngineConfig(threads=0), C)
    with pytest.raises(d3.ResourceError):
        d3.join_project(d3.RawTable(*r), d3.RawTable(*s),
                        d3.EngineConfig(force=d3.Strategy.hybrid, memory_budget_bytes=1024), C)


def _golden():
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_baseline_config_matches_reference(cfg):
    """Full BASELINE configs: count and (sum, xor) fingerprint of the distinct
    (x, z) set equal the reference's (tests/golden/golden.json), plus the
    dense/sparse split and exact OUT_J."""
    g = _golden().get(f"cfg{cfg}")
    if g is None:
        pytest.skip("golden entry not generated")
    rl, rr = d3.generate(cfg, 0)
    sl, sr = d3.generate(cfg, 1)
    # cfg3 is f1-gated to the classical join under auto (covered below); the
    # pipeline statistics of the golden record come from the DIM3 pipeline
    force = d3.Strategy.hybrid if cfg == 3 else d3.Strategy.auto_select
    out = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr),
                          d3.EngineConfig(force=force, count_only=True,
                                          checksum=True, memory_budget_bytes=64 << 30), C)
    rep = out.report
    assert rep.out_p == g["set"]["count"]
    assert rep.checksum_sum == g["set"]["sum"]
    assert rep.checksum_xor == g["set"]["xor"]
    p = g["pipeline"]
    for k in ("x_card", "y_card", "z_card", "r_nnz", "s_nnz", "out_j", "dense_z", "sparse_z",
              "sparse_nnz", "dropped_r"):
        assert getattr(rep, k) == p[k], k
    ref = g.get("ref_hybrid_report")
    if ref and cfg != 3:  # the reference's own pairs split (cfg2 folds its sparse rows)
        assert (rep.pairs_sparse, rep.pairs_dense) == (ref["pairs_sparse"], ref["pairs_dense"])


def test_cfg5_x_slice_matches_reference():
    """cfg5 (200M x 200M, Zipf 1.2): R restricted to x < 1000 against the full S
    (the engine swaps). Count, set fingerprint and per-100-x block
    fingerprints equal the reference's (tests/golden)."""
    import torch
    g = _golden().get("cfg5_x_lt_1000")
    if g is None:
        pytest.skip("golden entry not generated")
    rl, rr = d3.generate(5, 0)
    keep = rl < 1000
    rl, rr = rl[keep].contiguous(), rr[keep].contiguous()
    del keep
    sl, sr = d3.generate(5, 1)
    out = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr),
                          d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True,
                                          checksum=True, memory_budget_bytes=120 << 30), C)
    rep = out.report
    assert rep.swapped
    assert rep.out_p == g["set"]["count"] == 9976370095
    assert rep.checksum_sum == g["set"]["sum"]
    assert rep.checksum_xor == g["set"]["xor"]
    # per-block: the caller x of this slice spans [0, 1000); check block 0 (x < 100)
    blk = g["blocks"]
    rb = rl < 100
    o0 = d3.join_project(d3.RawTable(rl[rb].contiguous(), rr[rb].contiguous()), d3.RawTable(sl, sr),
                         d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True,
                                         checksum=True, memory_budget_bytes=120 << 30), C)
    assert (o0.report.out_p, o0.report.checksum_sum, o0.report.checksum_xor) == \
        (blk["count"][0], blk["sum"][0], blk["xor"][0])
    del rl, rr, sl, sr
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", [1, 2])
def test_tcgen05_hot_pass_matches_bit_sliced(cfg, monkeypatch):
    """The tcgen05 kind::i8 hot pass (comparison kernel) counts exactly the
    same dense pairs as the bit-sliced default."""
    rl, rr = d3.generate(cfg, 0)
    sl, sr = d3.generate(cfg, 1)
    e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True, memory_budget_bytes=64 << 30)
    monkeypatch.delenv("D3G_HOT", raising=False)
    a = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    monkeypatch.setenv("D3G_HOT", "tc")
    b = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    assert (a.out_p, a.pairs_dense, a.pairs_sparse) == (b.out_p, b.pairs_dense, b.pairs_sparse)


def _bag(r, s):
    """oracle_out_j_bag (P/tests/support.hpp:74-84)."""
    ys, cnt = np.unique(s[1], return_counts=True)
    d = dict(zip(ys.tolist(), cnt.tolist()))
    return int(sum(d.get(y, 0) for y in r[1].tolist()))


@pytest.mark.parametrize("variant", ["partitioned", "global"])
def test_classical_branch_matches_reference(variant, monkeypatch):
    """force=classical (hash_join_dedup, P/src/classical.cpp:111-210): same set,
    intermediate_pairs = the bag join size, strategy named in the report. Both
    GPU variants: x-partitioned (default) and the global pair-set dedup."""
    if variant == "global":
        monkeypatch.setenv("D3G_CLASSICAL", "global")
    else:
        monkeypatch.delenv("D3G_CLASSICAL", raising=False)
    rng = SplitMix64(503)
    for _ in range(10):
        r, s = random_instance(rng)
        out = _run(r, s, d3.Strategy.classical)
        assert out.report.strategy == "classical"
        assert pair_set(out.result.raw_x, out.result.raw_z) == oracle_pairs(r, s)
        big, small = (r, s) if len(r[0]) >= len(s[0]) else (s, r)
        assert out.report.intermediate_pairs == _bag(big, small)
        assert out.report.pairs_classical == out.report.out_p


def test_auto_gate_takes_classical_on_cfg3():
    """cfg3 has f1 = +15.67 > 0: auto runs the classical join, like
    the reference, and still produces the reference's set."""
    g = _golden()["cfg3"]
    rl, rr = d3.generate(3, 0)
    sl, sr = d3.generate(3, 1)
    out = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr),
                          d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True,
                                          checksum=True, memory_budget_bytes=64 << 30), C)
    rep = out.report
    assert rep.strategy == "classical" and rep.f1_gate_classical and rep.f1_value > 0
    assert (rep.out_p, rep.checksum_sum, rep.checksum_xor) == \
        (g["set"]["count"], g["set"]["sum"], g["set"]["xor"])


def test_classical_variants_agree_on_cfg3(monkeypatch):
    """The global-set and x-partitioned classical variants give the same count,
    fingerprint and bag join size on the full cfg3 workload."""
    rl, rr = d3.generate(3, 0)
    sl, sr = d3.generate(3, 1)
    e = d3.EngineConfig(force=d3.Strategy.classical, count_only=True, checksum=True,
                        memory_budget_bytes=64 << 30)
    monkeypatch.delenv("D3G_CLASSICAL", raising=False)
    a = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    monkeypatch.setenv("D3G_CLASSICAL", "global")
    b = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    assert a.strategy == b.strategy == "classical"
    assert (a.out_p, a.checksum_sum, a.checksum_xor, a.intermediate_pairs) == \
        (b.out_p, b.checksum_sum, b.checksum_xor, b.intermediate_pairs)
    assert a.pairs_classical == a.out_p


@pytest.mark.parametrize("cold", ["hash", "tiers"])
def test_cfg5_full_pipeline_x_range_matches_reference(cold, monkeypatch):
    """Full cfg5 (200M x 200M, no swap, 9,993,304 dense z as in the reference)
    with the kernels restricted to x codes [0, 1000) and to 100-x blocks: the
    pairs of those x are exactly the reference's x<1000 slice set (golden).
    Exercises the hash-deduplicated cold pass (10M dense rows) and, for
    comparison, the SparseBMM-tier cold pass."""
    import torch
    g = _golden().get("cfg5_x_lt_1000")
    if g is None:
        pytest.skip("golden entry not generated")
    if cold == "tiers":
        monkeypatch.setenv("D3G_COLD", "tiers")
    else:
        monkeypatch.delenv("D3G_COLD", raising=False)
    rl, rr = d3.generate(5, 0)
    sl, sr = d3.generate(5, 1)

    def run(lo, hi):
        e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True, checksum=True,
                            memory_budget_bytes=120 << 30, x_code_range=(lo, hi))
        return d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report

    rep = run(0, 1000)
    assert not rep.swapped and rep.dense_z == 9993304 and rep.sparse_z == 6696
    assert (rep.out_p, rep.checksum_sum, rep.checksum_xor) == \
        (g["set"]["count"], g["set"]["sum"], g["set"]["xor"])
    blk = g["blocks"]
    for b in (0, 9):
        r = run(100 * b, 100 * (b + 1))
        assert (r.out_p, r.checksum_sum, r.checksum_xor) == \
            (blk["count"][b], blk["sum"][b], blk["xor"][b])
    del rl, rr, sl, sr
    torch.cuda.empty_cache()


def test_self_join_reuses_the_csr_and_matches(monkeypatch):
    """S element-wise identical to R (cfg2's S := R): the engine builds the
    CSR once; sets, split and report equal the general path and the oracle
    (dictionary and natural keys)."""
    rng = SplitMix64(513)
    for _ in range(6):
        r, _s = random_instance(rng)
        s = (r[0].copy(), r[1].copy())
        want = oracle_pairs(r, s)
        monkeypatch.delenv("D3G_NO_SELFJOIN", raising=False)
        a = _run(r, s, d3.Strategy.hybrid)
        monkeypatch.setenv("D3G_NO_SELFJOIN", "1")
        b = _run(r, s, d3.Strategy.hybrid)
        assert pair_set(a.result.raw_x, a.result.raw_z) == want
        for k in ("out_p", "pairs_dense", "pairs_sparse", "dense_z", "s_nnz", "r_nnz", "out_j"):
            assert getattr(a.report, k) == getattr(b.report, k), k
        # the same host relation passed as both sides is copied to the device once
        t = d3.RawTable(*r)
        c = d3.join_project(t, t, d3.EngineConfig(force=d3.Strategy.hybrid), C)
        assert c.report.h2d_bytes == 16 * len(r[0])
        assert pair_set(c.result.raw_x, c.result.raw_z) == want


def test_rank0_split_count_only_cfg2(monkeypatch):
    """Count-only runs split the live x by the top-ranked y: pairs of x and z
    that both hold it are counted without a test. cfg2 at full size: the
    count and the reference's pairs_sparse/pairs_dense split are unchanged,
    with and without the split (D3G_NO_SPLIT)."""
    g = _golden()["cfg2"]
    ref = g["ref_hybrid_report"]
    rl, rr = d3.generate(2, 0)
    sl, sr = d3.generate(2, 1)
    e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True,
                        memory_budget_bytes=64 << 30)
    a = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    assert a.hot_direct_pairs > 0
    assert a.out_p == g["set"]["count"]
    assert (a.pairs_sparse, a.pairs_dense) == (ref["pairs_sparse"], ref["pairs_dense"])
    # one to six pivots (2 to 64 classes; class-aligned batches)
    for piv in ("1", "2", "3", "4", "5", "6"):
        monkeypatch.setenv("D3G_PIVOTS", piv)
        p = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
        assert p.hot_direct_pairs > 0, piv
        assert (p.out_p, p.pairs_sparse, p.pairs_dense) == (a.out_p, a.pairs_sparse, a.pairs_dense)
    monkeypatch.delenv("D3G_PIVOTS")
    monkeypatch.setenv("D3G_NO_SPLIT", "1")
    b = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    assert b.hot_direct_pairs == 0
    assert (b.out_p, b.pairs_sparse, b.pairs_dense) == (a.out_p, a.pairs_sparse, a.pairs_dense)


def test_rank0_split_count_only_cfg5_x_range():
    """cfg5 (200M x 200M) restricted to x codes [0, 300000): the split
    count-only run equals the checksum-mode run (which tests every pair)."""
    import torch
    rl, rr = d3.generate(5, 0)
    sl, sr = d3.generate(5, 1)

    def run(checksum):
        e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True, checksum=checksum,
                            memory_budget_bytes=120 << 30, x_code_range=(0, 300000))
        return d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report

    a, b = run(False), run(True)
    assert a.hot_direct_pairs > 0 and b.hot_direct_pairs == 0
    assert (a.out_p, a.pairs_sparse, a.pairs_dense) == (b.out_p, b.pairs_sparse, b.pairs_dense)
    del rl, rr, sl, sr
    torch.cuda.empty_cache()


def test_cfg5_cold_overflow_matches_reference(monkeypatch):
    """cfg5's hash cold pass with its per-warp limit forced down, so that most
    x overflow into the flattened global-bitmap kernel: the x<1000 slice still
    equals the reference's."""
    import torch
    g = _golden().get("cfg5_x_lt_1000")
    if g is None:
        pytest.skip("golden entry not generated")
    monkeypatch.setenv("D3G_COLD_HASH_MAX", "64")
    rl, rr = d3.generate(5, 0)
    sl, sr = d3.generate(5, 1)
    e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True, checksum=True,
                        memory_budget_bytes=120 << 30, x_code_range=(0, 1000))
    rep = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    assert (rep.out_p, rep.checksum_sum, rep.checksum_xor) == \
        (g["set"]["count"], g["set"]["sum"], g["set"]["xor"])
    del rl, rr, sl, sr
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", [3, 4])
def test_count_only_matches_reference(cfg):
    """The count-only path (the bench's step: no fingerprint, the pivot plan
    where it applies, the jump-table hot kernel without the subset table on
    cfg4) gives the reference's count and pairs split."""
    g = _golden().get(f"cfg{cfg}")
    if g is None:
        pytest.skip("golden entry not generated")
    rl, rr = d3.generate(cfg, 0)
    sl, sr = d3.generate(cfg, 1)
    out = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr),
                          d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True,
                                          memory_budget_bytes=64 << 30), C)
    rep = out.report
    assert rep.out_p == g["set"]["count"]
    ref = g.get("ref_hybrid_report")
    if ref and cfg != 3:
        assert (rep.pairs_sparse, rep.pairs_dense) == (ref["pairs_sparse"], ref["pairs_dense"])


def test_cfg5_cold_overflow_tiers_match_reference(monkeypatch):
    """Both overflow tiers of the hash cold pass forced on the cfg5 slice: a
    tiny per-warp limit sends most x to the CTA-hash tier and a tiny CTA limit
    sends them on to the global-bitmap tier; the x<1000 slice still equals
    the reference's."""
    import torch
    g = _golden().get("cfg5_x_lt_1000")
    if g is None:
        pytest.skip("golden entry not generated")
    monkeypatch.setenv("D3G_COLD_HASH_MAX", "64")
    monkeypatch.setenv("D3G_COLD_CTA_MAX", "256")
    rl, rr = d3.generate(5, 0)
    sl, sr = d3.generate(5, 1)
    e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True, checksum=True,
                        memory_budget_bytes=120 << 30, x_code_range=(0, 1000))
    rep = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    assert (rep.out_p, rep.checksum_sum, rep.checksum_xor) == \
        (g["set"]["count"], g["set"]["sum"], g["set"]["xor"])
    del rl, rr, sl, sr
    torch.cuda.empty_cache()


@pytest.mark.parametrize("env", [
    {"D3G_COLD_STAR": "1"},                              # every star hands its x to the CTA tier
    {"D3G_COLD_STAR": "1", "D3G_COLD_CTA_MAX": "256"},   # ... and on to the bitmap tier
    {"D3G_COLD_STAR": "4000000000", "D3G_COLD_ROUTE": "4000000000"},  # no x routed by size
    {"D3G_COLD_STAR": "64", "D3G_COLD_HASH_MAX": "200"},
])
def test_cfg5_cold_star_segment_matches_reference(env, monkeypatch):
    """The star segment of the hash cold pass (each x's longest segment is
    looked up in the finished dedup set instead of inserted) in all three
    tiers: routing thresholds forced so that the star is resolved by the warp
    tier, the CTA tier and the bitmap tier; count and fingerprint of the cfg5
    x<1000 slice equal the reference's."""
    import torch
    g = _golden().get("cfg5_x_lt_1000")
    if g is None:
        pytest.skip("golden entry not generated")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rl, rr = d3.generate(5, 0)
    sl, sr = d3.generate(5, 1)
    e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True, checksum=True,
                        memory_budget_bytes=120 << 30, x_code_range=(0, 1000))
    rep = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    assert (rep.out_p, rep.checksum_sum, rep.checksum_xor) == \
        (g["set"]["count"], g["set"]["sum"], g["set"]["xor"])
    del rl, rr, sl, sr
    torch.cuda.empty_cache()


def test_byte_string_columns_match_integer_run():
    """ColumnType::bytes columns (relation.hpp:21, hash_bytes keys in the
    reference's dictionaries): each column role as byte strings, all of them,
    and y columns of different types. The pairs decode to the strings of the
    integer run's pairs, and counts, cards, split and dropped rows equal the
    integer run with dictionary coding (what the reference does for bytes)."""
    rng = SplitMix64(77)
    enc = lambda col: np.array([b"k%d" % (int(v) * 7919 % 100003) for v in col], dtype=object)
    for _ in range(6):
        r, s = random_instance(rng)
        want = oracle_pairs(r, s)
        base = _run(r, s, d3.Strategy.hybrid, natural_keys_auto=False).report
        for variant in range(4):
            bx, by, bz = variant in (0, 3), variant in (1, 3), variant in (2, 3)
            rt = d3.RawTable(enc(r[0]) if bx else r[0], enc(r[1]) if by else r[1])
            st = d3.RawTable(enc(s[0]) if bz else s[0], enc(s[1]) if by else s[1])
            for f in (d3.Strategy.hybrid, d3.Strategy.auto_select, d3.Strategy.classical):
                out = d3.join_project(rt, st, d3.EngineConfig(force=f), C)
                got = set(zip(out.result.raw_x.tolist(), out.result.raw_z.tolist()))
                ex = {(enc([x])[0] if bx else x, enc([z])[0] if bz else z) for x, z in want}
                assert got == ex and out.report.out_p == len(want)
                cnt = d3.join_project(rt, st, d3.EngineConfig(force=f, count_only=True), C)
                assert cnt.report.out_p == len(want)
            rep = d3.join_project(rt, st, d3.EngineConfig(force=d3.Strategy.hybrid), C).report
            # (flags in engine orientation: the larger table's left column is x)
            sw = rep.swapped
            assert not (rep.natural_x and (bz if sw else bx))
            assert not (rep.natural_z and (bx if sw else bz)) and not (rep.natural_y and by)
            if variant == 3:
                assert (rep.x_card, rep.y_card, rep.z_card, rep.dense_z, rep.sparse_z,
                        rep.dropped_r, rep.pairs_dense, rep.pairs_sparse) == \
                    (base.x_card, base.y_card, base.z_card, base.dense_z, base.sparse_z,
                     base.dropped_r, base.pairs_dense, base.pairs_sparse)
        # y columns of different types: no R row finds its y
        rt = d3.RawTable(r[0], enc(r[1]))
        out = d3.join_project(rt, d3.RawTable(*s), d3.EngineConfig(force=d3.Strategy.hybrid), C)
        assert out.report.out_p == 0 and len(out.result.raw_x) == 0
        assert out.report.dropped_r == max(len(r[0]), len(s[0]))
        # declaring a byte-string column natural: the reference's ConfigError
        # (raised by map_tables, which the classical branch never calls)
        flags = d3.SkipFlags(y=True)
        rb, sb = d3.RawTable(r[0], enc(r[1])), d3.RawTable(s[0], enc(s[1]))
        with pytest.raises(d3.ConfigError):
            d3.join_project(rb, sb, d3.EngineConfig(force=d3.Strategy.hybrid,
                                                    natural_keys_declared=flags), C)
        out = d3.join_project(rb, sb, d3.EngineConfig(force=d3.Strategy.classical,
                                                      natural_keys_declared=flags), C)
        assert out.report.out_p == len(want)


@pytest.mark.parametrize("seed", [11, 12])
def test_hash_cold_pass_long_rows_match_bitmap_path(seed, monkeypatch):
    """The hash cold pass forced (D3G_COLD_PATH=hash) on skewed instances whose
    x rows hold 50-150 y values (several 32-row chunks per x: the star segment
    is the longest of the LAST chunk) gives the pairs, count and fingerprint
    of the bitmap cold kernel and of numpy; also with tiny tier limits."""
    rng = np.random.default_rng(seed)
    nx, ny, n = int(rng.integers(1200, 1800)), int(rng.integers(20000, 40000)), 120000
    w = 1.0 / np.arange(1, ny + 1) ** float(rng.uniform(0.6, 0.8))
    w /= w.sum()
    r = (rng.integers(0, nx, n).astype(np.uint64), rng.choice(ny, n, p=w).astype(np.uint64))
    s = (rng.integers(0, 4 * nx, n).astype(np.uint64), rng.choice(ny, n, p=w).astype(np.uint64))
    base = _run(r, s, d3.Strategy.hybrid, count_only=True, checksum=True).report
    # numpy: distinct (x, z) of the join, packed x << 32 | z
    ru = np.unique(np.stack(r, 1), axis=0)
    su = np.unique(np.stack(s, 1), axis=0)
    su = su[np.argsort(su[:, 1], kind="stable")]
    lo = np.searchsorted(su[:, 1], ru[:, 1], "left")
    hi = np.searchsorted(su[:, 1], ru[:, 1], "right")
    reps = hi - lo
    xs = np.repeat(ru[:, 0], reps)
    idx = np.repeat(lo, reps) + (np.arange(reps.sum()) - np.repeat(np.cumsum(reps) - reps, reps))
    want = np.unique((xs << np.uint64(32)) | su[idx, 0])
    assert base.out_p == len(want)
    assert base.cold_candidates > 0  # the cold pass has work
    for env in ({}, {"D3G_COLD_HASH_MAX": "32"},
                {"D3G_COLD_HASH_MAX": "32", "D3G_COLD_CTA_MAX": "64"}, {"D3G_COLD_STAR": "8"}):
        monkeypatch.setenv("D3G_COLD_PATH", "hash")
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        rep = _run(r, s, d3.Strategy.hybrid, count_only=True, checksum=True).report
        assert (rep.out_p, rep.checksum_sum, rep.checksum_xor) == \
            (base.out_p, base.checksum_sum, base.checksum_xor), env
        cnt = _run(r, s, d3.Strategy.hybrid, count_only=True).report
        assert cnt.out_p == base.out_p, env
        out = _run(r, s, d3.Strategy.hybrid)
        got = np.sort((np.asarray(out.result.raw_x, dtype=np.uint64) << np.uint64(32)) |
                      np.asarray(out.result.raw_z, dtype=np.uint64))
        assert np.array_equal(got, want), env
        for k in env:
            monkeypatch.delenv(k)


@pytest.mark.parametrize("seed", [7, 8, 9])
def test_pivot_plan_mid_size_instances(seed, monkeypatch):
    """Mid-size skewed instances (x over 20-40k, Zipf y over a few hundred
    values) where the pivot plan engages with mixed and pure batches: the
    count-only count and pairs split equal the checksum-mode run (every pair
    tested) for one to six pivots, in both orientations; and with the
    class-aligned batches switched off (D3G_NO_PAD: mixed batches)."""
    rng = np.random.default_rng(seed)
    nx, ny, n = int(rng.integers(20000, 40000)), int(rng.integers(200, 600)), 150000
    w = 1.0 / np.arange(1, ny + 1) ** float(rng.uniform(0.9, 1.3))
    w /= w.sum()
    r = (rng.integers(0, nx, n).astype(np.uint64), rng.choice(ny, n, p=w).astype(np.uint64))
    s = (rng.integers(0, nx // 2, n // 2).astype(np.uint64),
         rng.choice(ny, n // 2, p=w).astype(np.uint64))
    direct = 0
    for a, b in ((r, s), (s, r)):
        base = _run(a, b, d3.Strategy.auto_select, count_only=True, checksum=True).report
        for piv in ("1", "2", "3", "4", "5", "6"):
            monkeypatch.setenv("D3G_PIVOTS", piv)
            got = _run(a, b, d3.Strategy.auto_select, count_only=True).report
            assert (got.out_p, got.pairs_sparse, got.pairs_dense) == \
                (base.out_p, base.pairs_sparse, base.pairs_dense), (seed, piv)
            direct += got.hot_direct_pairs
        monkeypatch.setenv("D3G_NO_PAD", "1")
        got = _run(a, b, d3.Strategy.auto_select, count_only=True).report
        assert (got.out_p, got.pairs_sparse, got.pairs_dense) == \
            (base.out_p, base.pairs_sparse, base.pairs_dense), (seed, "mixed")
        monkeypatch.delenv("D3G_NO_PAD")
        monkeypatch.delenv("D3G_PIVOTS")
    assert direct > 0  # the plan engaged


def test_pivot_plan_with_nothing_left_to_test():
    """Every x and every z hold the two top-ranked y (plus a few others): the
    pivot plan answers every pair without a test (zero units for the hot
    kernel); the count equals the checksum-mode run and |X| * |Z|."""
    rng = np.random.default_rng(11)
    nx, nz, extra = 9000, 7000, 40
    def rel(n, keys):
        a = np.concatenate([np.arange(n), np.arange(n), np.arange(n)]).astype(np.uint64)
        b = np.concatenate([np.zeros(n), np.ones(n), 2 + rng.integers(0, extra, n)]).astype(np.uint64)
        return a, b
    r, s = rel(nx, 0), rel(nz, 1)
    base = _run(r, s, d3.Strategy.auto_select, count_only=True, checksum=True).report
    got = _run(r, s, d3.Strategy.auto_select, count_only=True).report
    assert base.out_p == nx * nz
    assert (got.out_p, got.pairs_sparse, got.pairs_dense) == \
        (base.out_p, base.pairs_sparse, base.pairs_dense)
    assert got.pairs_dense > 0 and got.hot_direct_pairs == got.pairs_dense  # all untested


def test_int32_columns_match_u64(monkeypatch):
    """d3g_table.value_bytes = 4 (the int32 workloads): uint32 host columns and
    int32 device tensors give the same sets and reports as u64 columns, with
    half the host->device bytes."""
    import torch
    rng = SplitMix64(611)
    for _ in range(8):
        r, s = random_instance(rng)
        if max(int(r[0].max(initial=0)), int(r[1].max(initial=0)), int(s[0].max(initial=0)),
               int(s[1].max(initial=0))) >= (1 << 32):
            continue
        a = _run(r, s, d3.Strategy.auto_select)
        r32 = tuple(np.asarray(c, np.uint32) for c in r)
        s32 = tuple(np.asarray(c, np.uint32) for c in s)
        b = _run(r32, s32, d3.Strategy.auto_select)
        assert pair_set(a.result.raw_x, a.result.raw_z) == pair_set(b.result.raw_x, b.result.raw_z)
        assert (a.report.out_p, a.report.dense_z, a.report.strategy) == \
            (b.report.out_p, b.report.dense_z, b.report.strategy)
        assert b.report.h2d_bytes * 2 == a.report.h2d_bytes
    g = [O.gen(1, 0).left, O.gen(1, 0).right, O.gen(1, 1).left, O.gen(1, 1).right]
    dev = [torch.from_numpy(c.astype(np.int32)).cuda() for c in g]
    out = d3.join_project(d3.RawTable(dev[0], dev[1]), d3.RawTable(dev[2], dev[3]),
                          d3.EngineConfig(force=d3.Strategy.hybrid, count_only=True,
                                          checksum=True), C).report
    assert (out.out_p, out.checksum_sum, out.checksum_xor) == \
        (9429141, 0x6F2F5D2033C05DA4, 0x50CAA74071957968)
    assert out.h2d_bytes == 0
