"""Reference-equivalent work counters at the boundary: DenseEcStats
(P/include/dim3/denseec.hpp:20-29, counted at P/src/denseec.cpp:46-64) under
every DensePathMode, and SpaStats::spa_allocations / spa_entries
(P/include/dim3/sparsebmm.hpp:15-19, P/src/sparsebmm.cpp:17-21). The GPU
report must carry exactly what the unmodified reference library reports for
the same input, constants, mode and thread count."""
import json
import os

import numpy as np
import pytest

import paper_2206_04995_b200 as d3
from oracle import oracle as O
from support import SplitMix64, random_instance

pytestmark = pytest.mark.gpu
C = d3.CostConstants.test_consts()
DENSE = ("dense_wide_encounters", "dense_probe_encounters", "dense_blocks_checked",
         "dense_probes_done", "dense_row_bitmaps_built")
MODES = {"cost_based": d3.DensePathMode.cost_based, "force_wide": d3.DensePathMode.force_wide,
         "force_probe": d3.DensePathMode.force_probe}


def _golden():
    p = os.path.join(os.path.dirname(__file__), "golden", "golden.json")
    return json.load(open(p))


@pytest.mark.parametrize("seed", [41, 201, 501])
@pytest.mark.parametrize("mode", list(MODES))
def test_dense_counters_match_reference_on_corpora(seed, mode):
    """Random instances of the reference's own generator: every DenseEC
    counter equals the reference's under each DensePathMode, with and
    without the per-pair pass (encounters and row bitmaps are always filled)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = SplitMix64(seed)
    for _ in range(8):
        r, s = random_instance(rng)
        for force in ("hybrid", "dense"):
            want = O.ref_join_project(O.Table(*r), O.Table(*s), force=force, threads=1,
                                      dense_mode=mode)
            f = d3.Strategy.hybrid if force == "hybrid" else d3.Strategy.dense_only
            cfg = d3.EngineConfig(force=f, count_only=True, dense_mode=MODES[mode],
                                  collect_counters=True)
            got = d3.join_project(d3.RawTable(*r), d3.RawTable(*s), cfg, C).report
            assert got.out_p == want["out_p"]
            for k in DENSE:
                assert getattr(got, k) == want[k], (k, mode, force)
            cfg.collect_counters = False
            lite = d3.join_project(d3.RawTable(*r), d3.RawTable(*s), cfg, C).report
            for k in ("dense_wide_encounters", "dense_probe_encounters",
                      "dense_row_bitmaps_built"):
                assert getattr(lite, k) == want[k], (k, mode, force)
            assert lite.dense_blocks_checked == lite.dense_probes_done == 0


@pytest.mark.parametrize("threads", [1, 4, 7])
def test_spa_counters_match_reference(threads):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = SplitMix64(301)
    for _ in range(6):
        r, s = random_instance(rng)
        want = O.ref_join_project(O.Table(*r), O.Table(*s), force="hybrid", threads=threads)
        got = d3.join_project(d3.RawTable(*r), d3.RawTable(*s),
                              d3.EngineConfig(force=d3.Strategy.hybrid, count_only=True,
                                              threads=threads), C).report
        assert (got.spa_allocations, got.spa_entries) == \
            (want["spa_allocations"], want["spa_entries"])
        assert got.spa_inner_count == want["spa_inner_count"]
        kv = dict(got.to_kv())
        assert kv["spa_allocations"] == str(want["spa_allocations"])


@pytest.mark.parametrize("cfg", [1, 2])
def test_dense_counters_full_config_golden(cfg):
    """cfg1 / cfg2 at full size (cfg2: 3.93e10 encounters): the counters equal
    the reference hybrid run recorded in tests/golden (W_D of SURVEY 8(d):
    cfg2 blocks 89,748,060,931, probes 37,180,012,048)."""
    ref = _golden()[f"cfg{cfg}"]["ref_hybrid_report"]
    rl, rr = d3.generate(cfg, 0)
    sl, sr = d3.generate(cfg, 1)
    got = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr),
                          d3.EngineConfig(force=d3.Strategy.hybrid, count_only=True,
                                          collect_counters=True,
                                          memory_budget_bytes=64 << 30), C).report
    for k in DENSE:
        assert getattr(got, k) == ref[k], k
    assert got.out_p == ref["out_p"]


def test_dense_counters_sum_over_x_ranges():
    """Counters are over the x codes a call processes: x ranges add up."""
    rl, rr = d3.generate(1, 0)
    sl, sr = d3.generate(1, 1)
    e = dict(force=d3.Strategy.hybrid, count_only=True, collect_counters=True)
    full = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), d3.EngineConfig(**e), C)
    tot = {k: 0 for k in DENSE}
    lite = {k: 0 for k in DENSE}
    for lo, hi in ((0, 3000), (3000, 3001), (3001, 10000)):
        rep = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr),
                              d3.EngineConfig(x_code_range=(lo, hi), **e), C).report
        rep2 = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr),
                               d3.EngineConfig(x_code_range=(lo, hi), force=d3.Strategy.hybrid,
                                               count_only=True), C).report
        for k in DENSE:
            tot[k] += getattr(rep, k)
            lite[k] += getattr(rep2, k)
    for k in DENSE:
        assert tot[k] == getattr(full.report, k), k
    for k in ("dense_wide_encounters", "dense_probe_encounters", "dense_row_bitmaps_built"):
        assert lite[k] == getattr(full.report, k), k


def _ref_dense_counts(rx, panel_rows, y_card, w, mode):
    """The reference's run_chunk counting (P/src/denseec.cpp:22-64) restated
    in Python for small instances: per live x and panel row, wide iff
    m_z > threshold; blocks / probes up to the first hit."""
    n_blocks = (y_card + w - 1) // w
    out = dict(wide=0, probe=0, blocks=0, probes=0, bitmaps=0)
    for x in range(rx.n_rows):
        ys = rx.col[rx.row_ptr[x]:rx.row_ptr[x + 1]].tolist()
        if not ys or not panel_rows:
            continue
        thr = {"cost_based": d3.f3_threshold(len(ys), y_card, C), "force_wide": 0,
               "force_probe": None}[mode]
        built = False
        ysset = set(ys)
        for zs in panel_rows:
            wide = thr is not None and len(zs) > thr
            common = sorted(ysset & set(zs))
            if wide:
                built = True
                out["wide"] += 1
                out["blocks"] += common[0] // w + 1 if common else n_blocks
            else:
                out["probe"] += 1
                out["probes"] += ys.index(common[0]) + 1 if common else len(ys)
        out["bitmaps"] += built
    return out


def test_kernel_level_dense_ec_counters():
    """d3g_dense_ec_rows (dim3::dense_ec over a BitmapPanel) fills
    DenseEcStats as the reference's dense_ec does, for every mode."""
    rng = SplitMix64(73)
    for _ in range(4):
        xc, yc, zc = 1 + rng.bounded(300), 1 + rng.bounded(700), 1 + rng.bounded(300)
        nr, ns = 1 + rng.bounded(4000), 1 + rng.bounded(4000)
        codes = lambda n, k: np.array([rng.bounded(k) for _ in range(n)], np.uint32)
        rx = d3.build_csr(codes(nr, xc), codes(nr, yc), xc, yc)
        sz = d3.build_csr(codes(ns, zc), codes(ns, yc), zc, yc)
        words = ((yc + C.w - 1) // C.w * C.w) // 64
        rows = [z for z in range(zc) if sz.row_ptr[z + 1] > sz.row_ptr[z]]
        panel_rows = [sz.col[sz.row_ptr[z]:sz.row_ptr[z + 1]].tolist() for z in rows]
        blocks = np.zeros(len(rows) * words, np.uint64)
        for j, zs in enumerate(panel_rows):
            for y in zs:
                blocks[j * words + y // 64] |= np.uint64(1) << np.uint64(y % 64)
        for mode, m in MODES.items():
            _, _, st = d3.dense_ec(rx, np.array(rows, np.uint32), blocks, yc, C, m,
                                   materialize=False)
            want = _ref_dense_counts(rx, panel_rows, yc, C.w, mode)
            assert (st.wide_encounters, st.probe_encounters, st.blocks_checked,
                    st.probes_done, st.row_bitmaps_built) == \
                (want["wide"], want["probe"], want["blocks"], want["probes"], want["bitmaps"]), mode
