"""world_size-2 gloo tests of the x-sharded multi-GPU host logic (CPU only).

Each rank owns an x shard of R (S replicated). Through the same exchange
object the library's host-callback transport uses
(paper_2206_04995_b200.distributed.TorchExchange), the ranks perform the
library's exchange sequence for the f2 inputs (csrc/engine.cu degree_stats:
MAX of the largest m_x, SUM of the m_x histogram padded to it with entry 0
recomputed from the job's x card, SUM of dR(y)) and its tally fold (GATHER of
per-rank records, sums and xor). The job's inputs must yield exactly the
single-process decision table, and the per-shard results (intersection-free)
must add up to the full count and fingerprint."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O
from stats_util import f2_inputs
from support import SplitMix64, oracle_pairs, random_instance


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    import paper_2206_04995_b200 as d3
    from paper_2206_04995_b200.distributed import TorchExchange, x_range_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = TorchExchange(dist)
    C = d3.CostConstants.test_consts()
    out = []
    try:
        for (r, s) in cases:
            full = f2_inputs(r, s)
            x_card = full["x_card"]
            lo, hi = x_range_bounds(x_card, rank, world)
            shard = f2_inputs(r, s, x_filter=lambda v: lo <= v < hi)
            ymax = full["y_card"]
            # the library's sequence (engine.cu degree_stats, dist branch)
            mx = np.array([len(shard["mx_hist"]) - 1], np.uint64)
            ex(d3.EX_MAX_U64, mx)
            hmx = np.zeros(int(mx[0]) + 1, np.uint64)
            hmx[1:len(shard["mx_hist"])] = np.asarray(shard["mx_hist"], np.uint64)[1:]
            ex(d3.EX_SUM_U64, hmx)
            hmx[0] = x_card - int(hmx[1:].sum())
            dr = np.zeros(max(ymax, 1), np.uint32)
            for y, c in shard["dr"].items():
                dr[int(y)] = c
            ex(d3.EX_SUM_U32, dr)
            spairs = np.unique(np.stack([s[0], s[1]], 1), axis=0)
            ds = np.zeros(max(ymax, 1), np.uint64)
            for y, c in zip(*np.unique(spairs[:, 1], return_counts=True)):
                ds[int(y)] = c
            out_j = int(np.dot(dr.astype(object), ds.astype(object)))
            t_sh, _ = d3.f2_decide(hmx, full["mz_hist"], x_card, ymax, full["z_card"], out_j, C)
            t_full, _ = d3.f2_decide(full["mx_hist"], full["mz_hist"], full["x_card"],
                                     full["y_card"], full["z_card"], full["out_j"], C)
            same_table = (out_j == full["out_j"] and np.array_equal(t_sh, t_full) and
                          np.array_equal(hmx[1:], np.asarray(full["mx_hist"], np.uint64)[1:]))
            # per-shard distinct pairs (brute force on the shard's R rows)
            keep = (r[0] >= lo) & (r[0] < hi)
            pairs = oracle_pairs((r[0][keep], r[1][keep]), s)
            xs = np.array([p[0] for p in pairs], np.uint64)
            zs = np.array([p[1] for p in pairs], np.uint64)
            n, x, sm = O.set_fingerprint(xs, zs) if len(pairs) else (0, 0, 0)
            # the tally fold (engine.cu: GATHER of records, sum / xor on the host)
            rec = np.zeros(3 * world, np.uint64)
            rec[3 * rank:3 * rank + 3] = (n, sm, x)
            buf = rec.view(np.uint8)
            ex(d3.EX_GATHER, buf)
            rec = buf.view(np.uint64).reshape(world, 3)
            tot = (int(rec[:, 0].sum()), int(rec[:, 1].sum()) & ((1 << 64) - 1),
                   int(np.bitwise_xor.reduce(rec[:, 2])))
            out.append((same_table, tot))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _natural_cases():
    rng = SplitMix64(777)
    cases = []
    while len(cases) < 6:
        r, s = random_instance(rng, 200, 3000)
        if int(r[0].max()) < 2 * r[0].size and int(r[1].max()) < 2 * r[1].size and \
                int(s[0].max()) < 2 * s[0].size and int(s[1].max()) < 2 * s[1].size and \
                r[0].size >= s[0].size:
            cases.append((r, s))
    # plus a cfg1 slice with a real dense block
    r1, s1 = O.gen(1, 0, 0, 20000), O.gen(1, 1, 0, 20000)
    cases.append(((r1.left, r1.right), (s1.left, s1.right)))
    return cases


def test_gloo_two_ranks_shard_and_reduce():
    cases = _natural_cases()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, cases, q)) for rk in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (r, s) in enumerate(cases):
        want = oracle_pairs(r, s)
        xs = np.array([p[0] for p in want], np.uint64)
        zs = np.array([p[1] for p in want], np.uint64)
        n, x, sm = O.set_fingerprint(xs, zs)
        for rk in range(world):
            same_table, tot = res[rk][i]
            assert same_table, (i, rk)
            assert tot == (n, sm, x), (i, rk)


def _ops_worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    import paper_2206_04995_b200 as d3
    from paper_2206_04995_b200.distributed import TorchExchange

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _apply_ops(TorchExchange(dist), rank, world, d3)))
    finally:
        dist.destroy_process_group()


def _apply_ops(fn, rank, world, d3):
    """The four exchange ops on rank-dependent inputs (u64 wrap-around, u32,
    max, gather)."""
    a = np.array([(1 << 64) - 1 - rank, 5 + rank, 1 << 63], np.uint64)
    fn(d3.EX_SUM_U64, a)
    b = np.array([0xFFFFFFFF, rank], np.uint32)
    fn(d3.EX_SUM_U32, b)
    c = np.array([rank, 100 - rank, 7], np.uint64)
    fn(d3.EX_MAX_U64, c)
    g = np.zeros(4 * world, np.uint8)
    g[4 * rank:4 * rank + 4] = rank + 1
    fn(d3.EX_GATHER, g)
    return a.tolist(), b.tolist(), c.tolist(), g.tolist()


def _ops_expected(world):
    m = (1 << 64) - 1
    a = [sum(m - r for r in range(world)) & m, sum(5 + r for r in range(world)) & m,
         (world << 63) & m]
    b = [(world * 0xFFFFFFFF) & 0xFFFFFFFF, sum(range(world)) & 0xFFFFFFFF]
    c = [world - 1, 100, 7]
    g = [q + 1 for q in range(world) for _ in range(4)]
    return a, b, c, g


def test_exchange_ops_gloo_and_threads():
    """The host-callback transports agree with the ops' definitions: gloo
    processes (TorchExchange) and threads (ThreadExchange)."""
    import threading

    import paper_2206_04995_b200 as d3
    from paper_2206_04995_b200.distributed import ThreadExchange
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ops_worker, args=(rk, world, port, q)) for rk in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _ops_expected(world)
    for rk in range(world):
        assert tuple(res[rk]) == want
    for n in (2, 3):
        te = ThreadExchange(n)
        got = {}
        th = [threading.Thread(target=lambda r=r: got.__setitem__(r, _apply_ops(te.rank_fn(r), r, n, d3)))
              for r in range(n)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for r in range(n):
            assert tuple(got[r]) == _ops_expected(n)


def test_bench_gpus_flag_launches_one_rank_per_gpu():
    """`bench.py --gpus N` without torchrun re-launches itself with N ranks
    (torch.distributed.run on 127.0.0.1); N = 1 stays a single process."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    for n in (1, 2):
        p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(n),
                            "--dry-run"], capture_output=True, text=True, timeout=300, env=env)
        assert p.returncode == 0, p.stderr[-2000:]
        import re
        lines = [json.loads(m) for m in re.findall(r"\{[^{}]*\}", p.stdout)]
        assert sorted(d["rank"] for d in lines) == list(range(n))
        assert all(d["world"] == n for d in lines)
        if n > 1:
            assert all(d["nccl_debug"] == "INFO" for d in lines)
