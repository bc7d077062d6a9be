"""The x-sharded join_project through the library's own
exchange: N ranks, each with its own context, pass their x-shard of R and the
whole S; the library exchanges the f2 inputs and the tallies. Run on ONE GPU
with the ranks as threads (ThreadExchange: only host threads wait on one
another, no kernel waits for another rank's), and with a one-rank NCCL
communicator (the NCCL transport's code path). Every rank must report exactly
the unsharded job: count, fingerprint, split, cards, OUT_J; the union of the
ranks' materialized pairs is the oracle's set."""
import threading

import numpy as np
import pytest

import paper_2206_04995_b200 as d3
from oracle import oracle as O
from paper_2206_04995_b200.distributed import ThreadExchange, shard_mask
from support import SplitMix64, oracle_pairs, pair_set, random_instance

pytestmark = pytest.mark.gpu
C = d3.CostConstants.test_consts()
JOB_KEYS = ("out_p", "checksum_sum", "checksum_xor", "pairs_sparse", "pairs_dense", "dense_z",
            "sparse_z", "x_card", "y_card", "z_card", "out_j", "r_nnz", "s_nnz", "x_live",
            "f2_evaluations", "spa_inner_count", "dropped_r", "strategy", "natural_x",
            "natural_y", "natural_z", "r_rows", "s_rows",
            "dense_wide_encounters", "dense_probe_encounters", "dense_row_bitmaps_built")


def run_sharded(r, s, nranks, cfg, x_card=None, contexts=None):
    """One thread per rank; returns the per-rank JoinProjectOutputs."""
    ex = ThreadExchange(nranks)
    outs, errs = [None] * nranks, []
    ctxs = contexts or [d3.Context(0) for _ in range(nranks)]

    def rank_main(q):
        try:
            ctx = ctxs[q]
            ctx.set_exchange(nranks, q, ex.rank_fn(q))
            keep = shard_mask(r[0], q, nranks, x_card)
            rq = d3.RawTable(np.ascontiguousarray(r[0][keep]), np.ascontiguousarray(r[1][keep]))
            outs[q] = d3.join_project(rq, d3.RawTable(*s), cfg, C, ctx=ctx)
        except BaseException as e:  # noqa: BLE001
            errs.append((q, e, getattr(ctxs[q], "exchange_error", None)))
            ex.barrier.abort()
        finally:
            ctxs[q].clear_exchange()

    th = [threading.Thread(target=rank_main, args=(q,)) for q in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        # the first rank to fail aborts the barrier; the others then fail in
        # their exchange callback: report the root cause
        root = [e for e in errs if not isinstance(e[2], threading.BrokenBarrierError)]
        q, e, cb = (root or errs)[0]
        if isinstance(e, (d3.ConfigError, d3.ResourceError)) and len(root) == len(errs):
            raise e
        raise AssertionError(f"rank {q}: {e!r} (callback: {cb!r}); all: {errs!r}")
    return outs


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_sharded_ranks_report_the_job(nranks):
    rng = SplitMix64(900 + nranks)
    ctxs = [d3.Context(0) for _ in range(nranks)]
    done = 0
    while done < 8:
        r, s = random_instance(rng)
        if len(s[0]) > len(r[0]):
            continue
        done += 1
        for force in (d3.Strategy.auto_select, d3.Strategy.hybrid, d3.Strategy.dense_only,
                      d3.Strategy.sparse_only):
            cfg = d3.EngineConfig(force=force, checksum=True)
            full = d3.join_project(d3.RawTable(*r), d3.RawTable(*s), cfg, C)
            outs = run_sharded(r, s, nranks, cfg, contexts=ctxs)
            got = set()
            for q, o in enumerate(outs):
                for k in JOB_KEYS + ("out_j_estimate", "f1_value"):  # <= 65,536 rows: exact
                    assert getattr(o.report, k) == getattr(full.report, k), (k, q, force)
                assert o.report.nranks == nranks and o.report.rank == q
                part = pair_set(o.result.raw_x, o.result.raw_z)
                assert not (part & got)
                got |= part
            assert got == oracle_pairs(r, s)
            assert sum(o.report.rank_out_p for o in outs) == full.report.out_p


def test_sharded_requires_the_larger_table_sharded():
    rng = SplitMix64(5)
    while True:
        r, s = random_instance(rng)
        if len(s[0]) > 2 * len(r[0]) + 8:
            break
    with pytest.raises(d3.ConfigError):
        run_sharded(r, s, 2, d3.EngineConfig(count_only=True))


@pytest.mark.parametrize("cfg,nranks,by_range", [(2, 4, True), (4, 3, False), (1, 8, True)])
def test_sharded_baseline_configs(cfg, nranks, by_range):
    """cfg2 (x ranges, 4 ranks), cfg4 (dictionary keys, hash shards, 3 ranks),
    cfg1 (8 ranks): the job's count (and fingerprint) equal the golden values."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
    want = g[f"cfg{cfg}"]["set"]
    r, s = O.gen(cfg, 0), O.gen(cfg, 1)
    x_card = {1: 10_000, 2: 200_000}.get(cfg) if by_range else None
    e = d3.EngineConfig(count_only=True, checksum=cfg != 4, memory_budget_bytes=32 << 30)
    outs = run_sharded((r.left, r.right), (s.left, s.right), nranks, e, x_card=x_card)
    for o in outs:
        assert o.report.out_p == want["count"]
        if cfg != 4:
            assert (o.report.checksum_sum, o.report.checksum_xor) == (want["sum"], want["xor"])
    p = g[f"cfg{cfg}"]["pipeline"]
    for k in ("x_card", "y_card", "z_card", "r_nnz", "s_nnz", "out_j", "dense_z", "sparse_z"):
        assert getattr(outs[0].report, k) == p[k], k


def test_nccl_one_rank_transport():
    """A one-rank NCCL communicator drives the NCCL code path (allreduce /
    allgather on the context's stream); the job equals the unsharded call."""
    ctx = d3.Context(0)
    try:
        ctx.set_nccl(d3.nccl_unique_id(), 1, 0)
    except d3.ConfigError as e:
        pytest.skip(f"NCCL not loadable: {e}")
    r, s = O.gen(1, 0), O.gen(1, 1)
    e = d3.EngineConfig(force=d3.Strategy.hybrid, count_only=True, checksum=True)
    got = d3.join_project(d3.RawTable(r.left, r.right), d3.RawTable(s.left, s.right), e, C,
                          ctx=ctx).report
    full = d3.join_project(d3.RawTable(r.left, r.right), d3.RawTable(s.left, s.right), e, C).report
    for k in JOB_KEYS:
        assert getattr(got, k) == getattr(full, k), k
    assert got.nranks == 1
    ctx.clear_exchange()


@pytest.mark.parametrize("nranks", [2, 5])
def test_zsplit_dense_only_instances(nranks):
    """The z-split S side (csrc/zsplit.cuh): with every z dense the ranks build
    S-by-z, the dense lists, hot records and the cold CSR for their own z
    range and gather them; every rank reports the unsharded job and the
    ranks' pairs are the oracle's set."""
    rng = SplitMix64(4200 + nranks)
    ctxs = [d3.Context(0) for _ in range(nranks)]
    done = 0
    while done < 6:
        r, s = random_instance(rng)
        if len(s[0]) > len(r[0]):
            continue
        done += 1
        cfg = d3.EngineConfig(force=d3.Strategy.dense_only, checksum=True)
        full = d3.join_project(d3.RawTable(*r), d3.RawTable(*s), cfg, C)
        outs = run_sharded(r, s, nranks, cfg, contexts=ctxs)
        got = set()
        for q, o in enumerate(outs):
            if full.report.dense_z and full.report.x_live:
                assert o.report.zsplit, q
            for k in JOB_KEYS:
                assert getattr(o.report, k) == getattr(full.report, k), (k, q)
            got |= pair_set(o.result.raw_x, o.result.raw_z)
        assert got == oracle_pairs(r, s)


def test_zsplit_cfg2_folded_layout():
    """cfg2 sharded 4 ways takes the z-split with its sparse rows folded into
    the dense layout; count, fingerprint and the pairs_sparse / pairs_dense
    split equal the unsharded call, and the z-split's collectives are
    accounted (calls, link bytes)."""
    r, s = O.gen(2, 0), O.gen(2, 1)
    e = d3.EngineConfig(count_only=True, checksum=True, memory_budget_bytes=32 << 30)
    full = d3.join_project(d3.RawTable(r.left, r.right), d3.RawTable(s.left, s.right), e, C).report
    outs = run_sharded((r.left, r.right), (s.left, s.right), 4, e, x_card=200_000)
    for o in outs:
        assert o.report.zsplit
        assert o.report.exchange_calls > 0 and o.report.exchange_bus_bytes > 0
        for k in ("out_p", "checksum_sum", "checksum_xor", "pairs_sparse", "pairs_dense",
                  "dense_z", "sparse_z", "out_j", "s_nnz", "r_nnz"):
            assert getattr(o.report, k) == getattr(full, k), k


@pytest.mark.parametrize("nranks", [3, 8])
def test_zsplit_count_only_plan_and_pooled_class0(nranks):
    """Count-only sharded cfg2: the pivot plan runs on every rank (class-
    aligned batches) and the ranks' class-0 x (no pivot) are pooled into
    shared batches tested against row slices; the job's count equals the
    reference's."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
    r, s = O.gen(2, 0), O.gen(2, 1)
    e = d3.EngineConfig(count_only=True, memory_budget_bytes=32 << 30)
    outs = run_sharded((r.left, r.right), (s.left, s.right), nranks, e, x_card=200_000)
    for o in outs:
        assert o.report.zsplit
        assert o.report.out_p == g["cfg2"]["set"]["count"]
        assert o.report.hot_direct_pairs > 0  # the plan counted pairs without a test
    assert sum(o.report.rank_out_p for o in outs) == g["cfg2"]["set"]["count"]
