"""CPU suite for the product boundary: the C-ABI library loads without a GPU,
exports every symbol include/dim3_b200.h declares, fails loudly (no CPU
fallback) when no device exists, and its host-side policy (f1, f3 threshold,
f2 decisions from degree histograms) equals the reference's decisions."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2206_04995_b200 as d3
from oracle import oracle as O
from stats_util import f2_inputs
from support import SplitMix64, random_instance

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dim3_b200.h")
C = d3.CostConstants.test_consts()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(d3g_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(d3.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(d3.EXPORTED) == syms


def test_version_and_defaults():
    lib = d3.lib()
    assert b"sm_100a" in lib.d3g_version()


def test_no_silent_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(d3.Dim3Error):
        d3.Context(0)
    r = d3.RawTable([1, 2], [3, 4])
    with pytest.raises(d3.Dim3Error):
        d3.join_project(r, r, d3.EngineConfig(), C)


def test_threads_validated_before_any_device_work():
    r = d3.RawTable([1], [2])
    with pytest.raises(d3.ConfigError):
        d3.join_project(r, r, d3.EngineConfig(threads=0), C)


def test_f1_and_f3_threshold_match_oracle():
    L = O.orc_lib()
    oc = O.make_consts()
    for (a, b, j) in [(1000, 2000, 500), (10 ** 6, 10 ** 6, 1714285), (5, 7, 0), (1, 1, 10 ** 12)]:
        assert d3.f1(a, b, j, C) == L.orc_f1(a, b, j, oc)
    for y in (1, 64, 1000, 50000):
        for mx in (1, 2, 3, 7, 22, 45, 100):
            assert d3.f3_threshold(mx, y, C) == L.orc_f3_threshold(mx, y, oc)


def _dense_from_table(inp, table):
    mz_per_z = inp["m_z_by_raw"]
    return {z for z, m in mz_per_z.items() if m < len(table) and table[m]}


@pytest.mark.parametrize("seed", [101, 201, 41])
def test_f2_decisions_match_reference_partition(seed):
    """d3g_f2_decide on the degree histograms picks exactly the reference's
    dense z (partition_s_csr's panel.z_ids), on the reference test corpora."""
    rng = SplitMix64(seed)
    n = 0
    for _ in range(20):
        r, s = random_instance(rng, 128, 2000)
        inp = f2_inputs(r, s)
        table, ev = d3.f2_decide(inp["mx_hist"], inp["mz_hist"], inp["x_card"], inp["y_card"],
                                 inp["z_card"], inp["out_j"], C)
        got = _dense_from_table(inp, table)
        if O.ref_available():
            want = set(O.ref_pipeline(O.Table(*r), O.Table(*s))["dense_z_raw"].tolist())
        else:
            want = None
        o = O.orc_join_project(O.Table(*r), O.Table(*s), force="hybrid")
        assert len(got) == o["dense_z"]
        assert ev == o["f2_evaluations"]
        if want is not None:
            assert got == want
        n += len(got)
    assert n > 0  # the corpus exercises dense decisions


def test_f2_decisions_cfg1_and_cfg2():
    for cfg, want in ((1, 9888), (2, 196594)):
        r, s = O.gen(cfg, 0), O.gen(cfg, 1)
        inp = f2_inputs((r.left, r.right), (s.left, s.right))
        table, _ = d3.f2_decide(inp["mx_hist"], inp["mz_hist"], inp["x_card"], inp["y_card"],
                                inp["z_card"], inp["out_j"], C)
        assert int(sum(inp["mz_hist"][m] for m in range(1, len(table)) if table[m])) == want


def test_forced_partitions():
    r, s = O.gen(1, 0), O.gen(1, 1)
    inp = f2_inputs((r.left, r.right), (s.left, s.right))
    t, ev = d3.f2_decide(inp["mx_hist"], inp["mz_hist"], inp["x_card"], inp["y_card"],
                         inp["z_card"], inp["out_j"], C, force=d3.Strategy.sparse_only)
    assert not t.any() and ev == 0
    t, ev = d3.f2_decide(inp["mx_hist"], inp["mz_hist"], inp["x_card"], inp["y_card"],
                         inp["z_card"], inp["out_j"], C, force=d3.Strategy.dense_only)
    assert t[0] == 0 and all(t[m] == (inp["mz_hist"][m] > 0) for m in range(1, len(t)))


def test_raw_table_column_widths():
    """uint32 host columns keep their width (d3g_table.value_bytes = 4); other
    integer dtypes are widened to u64; mixed widths are a FormatError."""
    t = d3.RawTable(np.array([1, 2], np.uint32), np.array([3, 4], np.uint32))
    assert t.left.dtype == np.uint32 and t.right.dtype == np.uint32
    t = d3.RawTable(np.array([1, 2], np.int64), np.array([3, 4], np.int32))
    assert t.left.dtype == np.uint64 and t.right.dtype == np.uint64
    with pytest.raises(d3.FormatError):
        d3.RawTable(np.array([1, 2], np.uint32), np.array([3, 4], np.uint64))
    with pytest.raises(d3.FormatError):
        d3.RawTable(np.array([-1, 2], np.int64), np.array([3, 4], np.int64))


def test_byte_string_columns_are_interned():
    """ColumnType::bytes columns (relation.hpp:21) become surrogate ids with
    equal strings <-> equal ids; the y columns share one id space (disjoint
    ranges when their types differ) and the D3G_KEYS_BYTES_* flags follow the
    engine's orientation (the larger table's left column is x)."""
    from paper_2206_04995_b200 import engine as E
    r = d3.RawTable(np.array([b"a", b"b", b"a"], dtype=object), np.array([b"p", b"q", b"p"], dtype=object))
    s = d3.RawTable(np.array([5, 6], np.uint64), np.array([b"q", b"r"], dtype=object))
    assert r.has_bytes and s.has_bytes
    r2, s2, dec_x, dec_z, flags = E._intern_bytes(r, s)
    assert dec_z is None and dec_x[r2.left.astype(np.int64)].tolist() == [b"a", b"b", b"a"]
    assert r2.right[0] == r2.right[2] != r2.right[1] and r2.right[1] == s2.right[0]
    assert len({int(s2.right[1]), *r2.right.tolist()}) == 3
    assert s2.left.tolist() == [5, 6] and s2.left.dtype == np.uint64
    assert flags == E.KEYS_BYTES_X | E.KEYS_BYTES_Y
    # the larger table is the engine's R whichever argument it is: its left
    # column stays the engine's x
    _, _, _, _, flags = E._intern_bytes(s, r)
    assert flags == E.KEYS_BYTES_X | E.KEYS_BYTES_Y
    big = d3.RawTable(np.arange(4, dtype=np.uint64), np.array([b"p"] * 4, dtype=object))
    assert E._intern_bytes(r, big)[4] == E.KEYS_BYTES_Z | E.KEYS_BYTES_Y  # r is the engine's S
    assert E._intern_bytes(big, r)[4] == E.KEYS_BYTES_Z | E.KEYS_BYTES_Y
    # y columns of different types: disjoint ids
    s3 = d3.RawTable(np.array([5, 6], np.uint64), np.array([0, 1], np.uint64))
    r3, s4, _, _, flags = E._intern_bytes(r, s3)
    assert not set(r3.right.tolist()) & set(s4.right.tolist()) and flags & E.KEYS_BYTES_Y
    with pytest.raises(d3.FormatError):
        d3.RawTable(np.array([b"a", 3], dtype=object), np.array([1, 2], np.uint64))
    with pytest.raises(d3.ConfigError):
        E._table_struct(r)
