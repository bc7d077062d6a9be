"""CPU suite: the oracle (plain-C restatement) pinned against the reference
itself (oracle/_ref) and against known answers from the reference's own tests
and the golden fixtures. No GPU needed."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from support import SplitMix64, oracle_pairs, random_instance

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))
need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def T(a, b):
    return O.Table(np.asarray(a, np.uint64), np.asarray(b, np.uint64))


def test_generator_matches_splitmix_restatement():
    """Convention G == SplitMix64 draws in Python."""
    r = O.gen(1, 0, 0, 4)
    s = O.gen(1, 1, 0, 2)
    rng = SplitMix64(1)
    want = [(rng.bounded(10000), rng.bounded(1000)) for _ in range(4)]
    assert list(zip(r.left.tolist(), r.right.tolist())) == want
    for _ in range(2 * (100000 - 4)):
        rng.next()
    assert list(zip(s.left.tolist(), s.right.tolist())) == [(rng.bounded(10000), rng.bounded(1000))
                                                           for _ in range(2)]


def test_cfg1_golden():
    """cfg1 count 9,429,141, sum 0x6f2f5d2033c05da4, xor 0x50caa74071957968,
    9,888 dense z, 380,894,863 blocks checked by the reference DenseEC."""
    r, s = O.gen(1, 0), O.gen(1, 1)
    d = O.orc_join_project(r, s, force="hybrid", threads=4)
    assert d["out_p"] == 9429141
    assert d["checksum_sum"] == 0x6F2F5D2033C05DA4
    assert d["checksum_xor"] == 0x50CAA74071957968
    assert (d["dense_z"], d["sparse_z"]) == (9888, 112)
    assert d["dense_blocks_checked"] == 380894863 and d["dense_probes_done"] == 0
    g = GOLDEN["cfg1"]
    for k, v in g["pipeline"].items():
        if k in d:
            assert d[k] == v, k
    assert (g["set"]["count"], g["set"]["sum"], g["set"]["xor"]) == \
        (d["out_p"], d["checksum_sum"], d["checksum_xor"])


def test_cfg3_golden():
    r, s = O.gen(3, 0), O.gen(3, 1)
    d = O.orc_join_project(r, s, force="hybrid", threads=8)
    g = GOLDEN["cfg3"]
    assert d["out_p"] == g["set"]["count"] == 40003400
    assert d["checksum_sum"] == g["set"]["sum"] == 0x5C18BAB40FA898A8
    assert d["checksum_xor"] == g["set"]["xor"] == 0x606B7DA237895812
    assert d["f1"] > 0  # auto would take the classical join
    for k in ("x_card", "y_card", "z_card", "r_nnz", "s_nnz", "out_j", "dense_z", "sparse_z"):
        assert d[k] == g["pipeline"][k], k


def test_golden_counts_agree_with_survey():
    assert GOLDEN["cfg2"]["set"]["count"] == 38841784410
    assert GOLDEN["cfg4"]["set"]["count"] == 93102044842
    assert GOLDEN["cfg5_x_lt_1000"]["set"]["count"] == 9976370095
    assert GOLDEN["cfg2"]["pipeline"]["dense_z"] == 196594
    assert GOLDEN["cfg2"]["pipeline"]["out_j"] == 101333906309
    assert GOLDEN["cfg4"]["pipeline"]["out_j"] == 96809352500
    rep = GOLDEN["cfg2"]["ref_hybrid_report"]
    assert rep["dense_blocks_checked"] == 89748060931
    assert rep["dense_probes_done"] == 37180012048


@need_ref
@pytest.mark.parametrize("seed", [41, 201, 301, 501])
def test_oracle_equals_reference_on_corpus(seed):
    """The restatement reproduces the reference exactly: emission order, every
    report counter and the dense/sparse split, for every strategy."""
    rng = SplitMix64(seed)
    for _ in range(15):
        r, s = random_instance(rng)
        want = oracle_pairs(r, s)
        for force in ("hybrid", "sparse", "dense"):
            for mode in ("cost_based", "force_wide", "force_probe"):
                o = O.orc_join_project(T(*r), T(*s), force=force, dense_mode=mode,
                                       count_only=False, want_pairs=True)
                e = O.ref_join_project(T(*r), T(*s), force=force, dense_mode=mode,
                                       count_only=False, want_pairs=True)
                assert set(map(tuple, o["pairs"].tolist())) == want
                assert np.array_equal(o["pairs"], e["pairs"])  # same emission order
                for k in ("out_p", "pairs_sparse", "pairs_dense", "sparse_z", "dense_z",
                          "f2_evaluations", "dropped_r", "x_card", "y_card", "z_card",
                          "spa_inner_count", "dense_wide_encounters", "dense_probe_encounters",
                          "dense_blocks_checked", "dense_probes_done",
                          "dense_row_bitmaps_built", "out_j_estimate", "panel_bytes",
                          "checksum_sum", "checksum_xor"):
                    assert o[k] == e[k], (k, force, mode)
                assert o["f1"] == e["f1"]


@need_ref
def test_oracle_pipeline_matches_reference_cfg1():
    r, s = O.gen(1, 0), O.gen(1, 1)
    p = O.ref_pipeline(r, s)
    o = O.orc_join_project(r, s, force="hybrid")
    for k in ("x_card", "y_card", "z_card", "r_nnz", "s_nnz", "out_j", "dense_z", "sparse_z",
              "sparse_nnz", "dropped_r"):
        assert o[k] == p[k], k


def test_known_answers():
    # |OUT_P| = 4
    d = O.orc_join_project(T([0, 0, 1], [0, 1, 1]), T([0, 0, 1], [0, 1, 1]), force="sparse",
                           count_only=False, want_pairs=True)
    assert set(map(tuple, d["pairs"].tolist())) == {(0, 0), (0, 1), (1, 0), (1, 1)}
    assert d["spa_inner_count"] == 5  # |OUT_J| = 5
    # test_cli.cpp:67-84 fixture count 4
    d = O.orc_join_project(T([1, 1, 2], [10, 11, 10]), T([5, 6, 6], [10, 11, 10]), force="auto")
    assert d["out_p"] == 4
    # test_mapping.cpp:89-106: semi-join drops the R row whose y misses S
    big = 1 << 40
    d = O.orc_join_project(T([1 + big, 2 + big, 3 + big, 4 + big], [10 + big, 20 + big, 99 + big, 10 + big]),
                           T([7 + big, 8 + big], [10 + big, 20 + big]), force="hybrid")
    assert d["dropped_r"] == 1 and d["natural_y"] == 0
    # test_mapping.cpp:122-137: identity card = max + 1 across both tables, and
    # the y semi-join filter is off under identity codes (R's y=3 is kept)
    d = O.orc_join_project(T([3, 1, 0, 2], [1, 3, 0, 2]), T([2, 0], [1, 1]), force="hybrid")
    assert d["natural_y"] == 1 and d["y_card"] == 4 and d["dropped_r"] == 0


def test_costmodel_known_answers():
    L = O.orc_lib()
    c = O.make_consts()
    # f3 threshold separates the sign exactly (test_costmodel.cpp:192-200)
    for mx in range(1, 65):
        t = L.orc_f3_threshold(mx, 64, c)
        for mz in range(1, 65):
            assert (mz > t) == (L.orc_f3(mx, mz, 64, c) > 0)
    # bucket keys (test_costmodel.cpp:225-245)
    assert [L.orc_mx_bucket_key(m) for m in (1, 9, 10, 57, 99, 100, 999, 12345)] == \
        [1, 9, 11, 15, 19, 21, 29, 41]
    assert [L.orc_mz_bucket_index(a, b) for a, b in
            ((0, 100), (1, 100), (99, 100), (100, 100), (5, 1000), (10, 1000), (999, 1000), (0, 0))] == \
        [0, 1, 99, 99, 0, 1, 99, 0]
    # f1 closed form (test_costmodel.cpp:15-32)
    cc = O.make_consts(dict(O.TEST_CONSTS, t_map=30e-9, t_randRW=80e-9, t_hash=150e-9))
    assert L.orc_f1(1000, 2000, 500, cc) == pytest.approx(2.0 * 3000 * 30e-9 + 500 * (80e-9 - 150e-9))
    assert L.orc_f1(1000000, 1000000, 1714285, cc) > 0
    assert L.orc_f1(1000000, 1000000, 1714287, cc) < 0
