"""map_tables on the GPU (d3g_map_tables): the reference's known answers
(P/tests/test_mapping.cpp:89-140) and, on random instances with u64 keys and
semi-join drops, the EXACT codes, cards and r_kept of the unmodified
reference library."""
import numpy as np
import pytest

import paper_2206_04995_b200 as d3
from oracle import oracle as O
from support import SplitMix64

pytestmark = pytest.mark.gpu


def _t(rows):
    a = np.array([p[0] for p in rows], np.uint64)
    b = np.array([p[1] for p in rows], np.uint64)
    return d3.RawTable(a, b)


def test_semi_join_drops_and_r_kept():
    """test_mapping.cpp:89-106."""
    s = _t([(7, 10), (8, 20)])
    m = d3.map_tables(_t([(1, 10), (2, 20), (3, 99), (4, 10)]), s)
    assert m.dropped_r == 1 and m.r_a.size == 3
    assert m.r_kept.tolist() == [0, 1, 3]
    assert m.z_card == 2
    m2 = d3.map_tables(_t([(1, 10), (2, 20)]), s)
    assert m2.dropped_r == 0 and m2.r_kept.size == 0


def test_codes_decode_to_values():
    """test_mapping.cpp:108-121."""
    r = _t([(100, 10), (200, 20), (100, 20)])
    s = _t([(5000, 20), (6000, 10), (5000, 10)])
    m = d3.map_tables(r, s)
    assert m.rev_x[m.r_a].tolist() == [100, 200, 100]
    assert m.rev_y[m.r_b].tolist() == [10, 20, 20]
    assert m.rev_z[m.s_a].tolist() == [5000, 6000, 5000]
    assert m.rev_y[m.s_b].tolist() == [20, 10, 10]


def test_skip_flags_identity_and_no_filter():
    """test_mapping.cpp:123-140: identity codes, no semi-join under identity
    y, card = max over both tables + 1."""
    m = d3.map_tables(_t([(3, 7), (1, 9)]), _t([(2, 7), (0, 7)]),
                      d3.SkipFlags(x=True, y=True, z=True))
    assert m.dropped_r == 0
    assert m.r_a.tolist() == [3, 1] and m.r_b.tolist() == [7, 9]
    assert m.y_card == 10
    assert m.rev_x is None and m.rev_y is None and m.rev_z is None
    with pytest.raises(d3.ConfigError):
        d3.map_tables(_t([(1 << 33, 1)]), _t([(1, 1)]), d3.SkipFlags(x=True))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("mode", ["dict", "auto"])
def test_codes_equal_reference(mode):
    """Random u64 keys (dictionary path: codes from the (LLC partition, first
    occurrence) order of Dictionary::build_impl) and small natural keys
    (auto: map_with_fallback), with dropped R rows: identical codes."""
    rng = SplitMix64(611)
    for _ in range(8):
        nr, ns = 1 + rng.bounded(30000), 1 + rng.bounded(30000)
        big = mode == "dict"
        xs = [rng.next() if big else rng.bounded(2000) for _ in range(64 + rng.bounded(2000))]
        ys = [rng.next() if big else rng.bounded(3000) for _ in range(64 + rng.bounded(3000))]
        zs = [rng.next() if big else rng.bounded(2000) for _ in range(64 + rng.bounded(2000))]
        r = (np.array([xs[rng.bounded(len(xs))] for _ in range(nr)], np.uint64),
             np.array([ys[rng.bounded(len(ys))] for _ in range(nr)], np.uint64))
        s = (np.array([zs[rng.bounded(len(zs))] for _ in range(ns)], np.uint64),
             np.array([ys[rng.bounded(len(ys) // 2 + 1)] for _ in range(ns)], np.uint64))
        want = O.ref_map_tables(O.Table(*r), O.Table(*s), None if mode == "auto" else (0, 0, 0))
        got = d3.map_tables(d3.RawTable(*r), d3.RawTable(*s), natural_keys_auto=(mode == "auto"))
        for k in ("dropped_r", "x_card", "y_card", "z_card"):
            assert getattr(got, k) == want[k], k
        assert np.array_equal(got.r_a, want["r_a"]) and np.array_equal(got.r_b, want["r_b"])
        assert np.array_equal(got.s_a, want["s_a"]) and np.array_equal(got.s_b, want["s_b"])
        assert np.array_equal(got.r_kept, want["r_kept"])
