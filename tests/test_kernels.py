"""Kernel-level entry points of the C ABI (d3g_build_csr, d3g_sparse_bmm_csr,
d3g_dense_ec_rows) against direct restatements of the reference's
definitions on the reference's own random instances, plus the sharding
properties the multi-GPU path relies on (x-shards and x-code ranges
partition the output exactly)."""
import numpy as np
import pytest

import paper_2206_04995_b200 as d3
from support import SplitMix64, oracle_pairs, pair_set, random_instance

pytestmark = pytest.mark.gpu
C = d3.CostConstants.test_consts()


def _csr_np(a, b, a_card):
    """build_csr (P/src/relation.cpp:206-258): rows sorted, duplicates collapsed."""
    pairs = np.unique(np.stack([a.astype(np.uint64), b.astype(np.uint64)], axis=1), axis=0)
    rp = np.zeros(a_card + 1, np.uint64)
    np.add.at(rp, pairs[:, 0].astype(np.int64) + 1, 1)
    return np.cumsum(rp).astype(np.uint64), pairs[:, 1].astype(np.uint32)


def _codes(rng, n, card):
    return np.array([rng.bounded(card) for _ in range(n)], np.uint32)


def test_build_csr_collapses_and_sorts():
    """test_relation.cpp:149-171 (six tuples, one duplicate -> nnz 5) and
    random code columns in both orientations."""
    a = np.array([1, 1, 1, 0, 2, 2], np.uint32)
    b = np.array([7, 3, 7, 2, 9, 1], np.uint32)
    m = d3.build_csr(a, b, 3, 10)
    assert m.nnz() == 5
    assert m.row_ptr.tolist() == [0, 1, 3, 5] and m.col.tolist() == [2, 3, 7, 1, 9]
    rng = SplitMix64(77)
    for _ in range(6):
        ac, bc = 1 + rng.bounded(3000), 1 + rng.bounded(3000)
        n = 1 + rng.bounded(40000)
        a, b = _codes(rng, n, ac), _codes(rng, n, bc)
        for major_is_a in (True, False):
            got = d3.build_csr(a, b, ac, bc, major_is_a)
            rp, col = _csr_np(a, b, ac) if major_is_a else _csr_np(b, a, bc)
            assert np.array_equal(got.row_ptr, rp) and np.array_equal(got.col, col)


@pytest.mark.parametrize("path", ["bucket", "scatter"])
def test_build_csr_paths_match_definition(path, monkeypatch):
    """Both CSR builders (the bucketed shared-memory build and the per-row
    scatter + segmented sort) against the definition: uniform majors of
    several densities, long rows (> 256 entries: the rank-sort tier), heavy
    duplication, and a skewed major whose bucket overflows shared memory
    (the bucketed path hands it to the scatter path)."""
    monkeypatch.setenv("D3G_CSR", path)
    rs = np.random.default_rng(5)
    cases = []
    for ac, bc, n in ((1000, 5000, 300000), (70000, 1 << 20, 600000), (3, 100000, 200000),
                      (5000, 64, 400000), (1, 1, 10), (2000, 3000, 1)):
        cases.append((rs.integers(0, ac, n).astype(np.uint32),
                      rs.integers(0, bc, n).astype(np.uint32), ac, bc))
    # one row holds ~40% of the tuples: its bucket exceeds the smem capacity
    a = rs.integers(0, 20000, 500000).astype(np.uint32)
    a[: 200000] = 17
    cases.append((a, rs.integers(0, 1 << 20, 500000).astype(np.uint32), 20000, 1 << 20))
    for a, b, ac, bc in cases:
        got = d3.build_csr(a, b, ac, bc)
        rp, col = _csr_np(a, b, ac)
        assert np.array_equal(got.row_ptr, rp), (path, ac, bc, len(a))
        assert np.array_equal(got.col, col), (path, ac, bc, len(a))


def _random_csrs(rng):
    xc, yc, zc = 1 + rng.bounded(400), 1 + rng.bounded(400), 1 + rng.bounded(400)
    nr, ns = 1 + rng.bounded(8000), 1 + rng.bounded(8000)
    rx = d3.build_csr(_codes(rng, nr, xc), _codes(rng, nr, yc), xc, yc)
    sy = d3.build_csr(_codes(rng, ns, yc), _codes(rng, ns, zc), yc, zc)
    return rx, sy, xc, yc, zc


def _join_np(rx, sy, xc):
    out = set()
    for x in range(xc):
        for y in rx.col[rx.row_ptr[x]:rx.row_ptr[x + 1]].tolist():
            for z in sy.col[sy.row_ptr[y]:sy.row_ptr[y + 1]].tolist():
                out.add((x, z))
    return out


def test_sparse_bmm_matches_definition():
    """sparse_bmm (P/src/sparsebmm.cpp:53-106): each (x, z) once; the inner
    count is the reference's SpA body count (OUT_J restricted to the sparse
    side); count-only agrees with materialization (test_sparsebmm.cpp:75)."""
    rng = SplitMix64(78)
    for _ in range(8):
        rx, sy, xc, yc, zc = _random_csrs(rng)
        want = _join_np(rx, sy, xc)
        n, pairs, st = d3.sparse_bmm(rx, sy, zc)
        assert n == len(want) and set(map(tuple, pairs.tolist())) == want
        assert pairs.tolist() == sorted(pairs.tolist())  # (x, z) order
        dr = np.bincount(rx.col, minlength=yc)
        ds = np.diff(sy.row_ptr.astype(np.int64))
        assert st.inner_count == int((dr * ds).sum())
        n2, none, _ = d3.sparse_bmm(rx, sy, zc, materialize=False)
        assert n2 == n and none is None
    # empty inputs yield nothing (test_sparsebmm.cpp:137)
    e = d3.build_csr(np.zeros(0, np.uint32), np.zeros(0, np.uint32), 4, 4)
    assert d3.sparse_bmm(e, e, 4)[0] == 0


def test_dense_ec_matches_definition():
    """dense_ec (P/src/denseec.cpp:90-153) over a BitmapPanel: (x, z_ids[j])
    iff R[x] meets panel row j; every dense path mode gives the same pairs
    (test_denseec.cpp:56-100), and an empty panel emits nothing (:154)."""
    rng = SplitMix64(79)
    for _ in range(6):
        xc, yc, zc = 1 + rng.bounded(400), 1 + rng.bounded(400), 1 + rng.bounded(400)
        nr, ns = 1 + rng.bounded(8000), 1 + rng.bounded(8000)
        rx = d3.build_csr(_codes(rng, nr, xc), _codes(rng, nr, yc), xc, yc)
        sz = d3.build_csr(_codes(rng, ns, zc), _codes(rng, ns, yc), zc, yc)  # z-major over y
        w = C.w
        words = ((yc + w - 1) // w * w) // 64
        rows = [z for z in range(min(zc, 300)) if sz.row_ptr[z + 1] > sz.row_ptr[z]]
        blocks = np.zeros(len(rows) * words, np.uint64)
        for j, z in enumerate(rows):
            for y in sz.col[sz.row_ptr[z]:sz.row_ptr[z + 1]].tolist():
                blocks[j * words + y // 64] |= np.uint64(1) << np.uint64(y % 64)
        zids = np.array(rows, np.uint32)
        want = set()
        for x in range(xc):
            ys = set(rx.col[rx.row_ptr[x]:rx.row_ptr[x + 1]].tolist())
            for j, z in enumerate(rows):
                if ys & set(sz.col[sz.row_ptr[z]:sz.row_ptr[z + 1]].tolist()):
                    want.add((x, z))
        for mode in (d3.DensePathMode.cost_based, d3.DensePathMode.force_wide,
                     d3.DensePathMode.force_probe):
            n, pairs, _ = d3.dense_ec(rx, zids, blocks, yc, C, mode)
            assert n == len(want) and set(map(tuple, pairs.tolist())) == want
    n, _, _ = d3.dense_ec(rx, np.zeros(0, np.uint32), np.zeros(0, np.uint64), yc, C)
    assert n == 0


@pytest.mark.parametrize("shards", [2, 3, 5])
def test_x_shards_partition_the_output(shards):
    """The multi-GPU split (shard_index/shard_count): shard results are
    disjoint and their union is the full result, on random instances and on
    cfg2 (count + fingerprint)."""
    rng = SplitMix64(80 + shards)
    for _ in range(5):
        r, s = random_instance(rng)
        want = oracle_pairs(r, s)
        got = set()
        total = 0
        for i in range(shards):
            out = d3.join_project(d3.RawTable(*r), d3.RawTable(*s),
                                  d3.EngineConfig(shard_index=i, shard_count=shards), C)
            part = pair_set(out.result.raw_x, out.result.raw_z)
            assert not (part & got)
            got |= part
            total += out.report.out_p
        assert got == want and total == len(want)
    rl, rr = d3.generate(2, 0)
    sl, sr = d3.generate(2, 1)
    e = dict(count_only=True, checksum=True, memory_budget_bytes=16 << 30)
    full = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), d3.EngineConfig(**e), C).report
    cnt, sm, xr = 0, 0, 0
    for i in range(shards):
        rep = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr),
                              d3.EngineConfig(shard_index=i, shard_count=shards, **e), C).report
        cnt += rep.out_p
        sm = (sm + rep.checksum_sum) % (1 << 64)
        xr ^= rep.checksum_xor
    assert (cnt, sm, xr) == (full.out_p, full.checksum_sum, full.checksum_xor)


def test_x_code_ranges_partition_the_output():
    """x_code_range restricts the kernels to [lo, hi) of engine x codes;
    consecutive ranges partition the result (the contiguous-range sharding)."""
    rng = SplitMix64(90)
    for _ in range(6):
        r, s = random_instance(rng)
        want = oracle_pairs(r, s)
        hy = d3.Strategy.hybrid  # the classical report carries no code cards
        full = d3.join_project(d3.RawTable(*r), d3.RawTable(*s), d3.EngineConfig(force=hy), C)
        swapped = full.report.swapped
        xc = full.report.x_card
        cuts = sorted({0, xc, rng.bounded(xc + 1), rng.bounded(xc + 1)})
        got = set()
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            if lo == hi:
                continue
            out = d3.join_project(d3.RawTable(*r), d3.RawTable(*s),
                                  d3.EngineConfig(force=hy, x_code_range=(lo, hi)), C)
            part = pair_set(out.result.raw_x, out.result.raw_z)
            assert not (part & got)
            got |= part
        assert got == want, swapped
    with pytest.raises(d3.ConfigError):
        d3.join_project(d3.RawTable(*r), d3.RawTable(*s), d3.EngineConfig(x_code_range=(5, 2)), C)
