"""cfg5 (BASELINE configs[4]: R, S 200M tuples each, x, z ~ U[0, 1e7),
y ~ Zipf(1.2) over [0, 1e6), seed 5) -- the config the headline metric is
quoted on -- checked across its WHOLE x range:

* 24 reference-computed 100-x block fingerprints spread over [0, 1e7), the
  last block included (tests/golden/make_golden.py, key cfg5_blocks: R
  restricted to those blocks against the full S through the unmodified
  reference, pairs bucketed by raw x / 100);
* the default count-only plan over the full range (four pivots, the bench's
  step) against the every-pair-tested checksum mode;
* the sum of 8 x-shard fingerprints against the unsharded fingerprint
  (the multi-GPU split), and count-only shard counts against the total.
"""
import json
import os

import pytest

import paper_2206_04995_b200 as d3

pytestmark = pytest.mark.gpu
C = d3.CostConstants.test_consts()
M64 = (1 << 64) - 1


def _golden():
    p = os.path.join(os.path.dirname(__file__), "golden", "golden.json")
    return json.load(open(p))


@pytest.fixture(scope="module")
def cfg5():
    import torch
    rl, rr = d3.generate(5, 0)
    sl, sr = d3.generate(5, 1)
    yield d3.RawTable(rl, rr), d3.RawTable(sl, sr)
    del rl, rr, sl, sr
    torch.cuda.empty_cache()


def _run(tabs, **kw):
    e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True,
                        memory_budget_bytes=120 << 30, **kw)
    return d3.join_project(tabs[0], tabs[1], e, C).report


def test_cfg5_blocks_across_the_x_range(cfg5):
    g = _golden().get("cfg5_blocks")
    if g is None:
        pytest.skip("golden entry not generated")
    w = g["width"]
    assert g["blocks"][0] == 0 and g["blocks"][-1] == 10_000_000 // w - 1
    for b, cnt, sm, xr in zip(g["blocks"], g["count"], g["sum"], g["xor"]):
        rep = _run(cfg5, checksum=True, x_code_range=(b * w, (b + 1) * w))
        assert not rep.swapped and rep.dense_z == 9993304 and rep.sparse_z == 6696
        assert (rep.out_p, rep.checksum_sum, rep.checksum_xor) == (cnt, sm, xr), b


def test_cfg5_full_range_count_only_equals_every_pair_checksum(cfg5):
    """The bench's step (count-only: the pivot plan counts most pairs without
    a test) against the checksum mode, which tests every pair; the count and
    the reference's sparse/dense split (f2 on the whole job) agree."""
    a = _run(cfg5)
    assert a.hot_direct_pairs > 0
    b = _run(cfg5, checksum=True)
    assert b.hot_direct_pairs == 0
    assert (a.out_p, a.pairs_sparse, a.pairs_dense) == (b.out_p, b.pairs_sparse, b.pairs_dense)
    assert a.out_p == 99_739_429_407_838
    # the 8-way x-shard split (the multi-GPU partition): fingerprints add up
    cnt, sm, xr, cnt_only = 0, 0, 0, 0
    for i in range(8):
        r = _run(cfg5, checksum=True, shard_index=i, shard_count=8)
        cnt += r.out_p
        sm = (sm + r.checksum_sum) & M64
        xr ^= r.checksum_xor
        cnt_only += _run(cfg5, shard_index=i, shard_count=8).out_p
    assert (cnt, sm, xr) == (b.out_p, b.checksum_sum, b.checksum_xor)
    assert cnt_only == a.out_p


def test_cfg5_high_x_codes_partition(cfg5):
    """x codes near 1e7 (the last shard's end, the smallest-degree batches):
    contiguous x-code ranges at the top of the range add up to their union."""
    lo, mid, hi = 9_990_000, 9_999_950, 10_000_000
    u = _run(cfg5, checksum=True, x_code_range=(lo, hi))
    a = _run(cfg5, checksum=True, x_code_range=(lo, mid))
    b = _run(cfg5, checksum=True, x_code_range=(mid, hi))
    assert a.out_p + b.out_p == u.out_p > 0
    assert (a.checksum_sum + b.checksum_sum) & M64 == u.checksum_sum
    assert a.checksum_xor ^ b.checksum_xor == u.checksum_xor
