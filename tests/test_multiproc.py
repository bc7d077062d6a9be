"""world_size-2 gloo tests of the x-sharded multi-GPU host logic (CPU only).

Each rank owns an x shard of R (S replicated). The all-reduced f2 inputs must
yield exactly the single-process decision table, and the per-shard results
(intersection-free) must add up to the full count and fingerprint."""
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
    from paper_2206_04995_b200.distributed import allreduce_f2_inputs, reduce_tally, x_shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    C = d3.CostConstants.test_consts()
    out = []
    try:
        for (r, s) in cases:
            full = f2_inputs(r, s)
            x_card = full["x_card"]
            lo, hi = x_shard_bounds(x_card, rank, world)
            shard = f2_inputs(r, s, x_filter=lambda v: lo <= v < hi)
            ymax = full["y_card"]
            dr = np.zeros(max(ymax, 1), np.uint64)
            for y, c in shard["dr"].items():
                dr[int(y)] = c
            ds = np.zeros(max(ymax, 1), np.uint64)
            spairs = np.unique(np.stack([s[0], s[1]], 1), axis=0)
            for y, c in zip(*np.unique(spairs[:, 1], return_counts=True)):
                ds[int(y)] = c
            loc = {"mx_hist": shard["mx_hist"], "dr": dr, "x_card": x_card,
                   "r_nnz": int(sum(m * int(c) for m, c in enumerate(shard["mx_hist"]))),
                   "mz_hist": full["mz_hist"], "ds": ds, "y_card": ymax,
                   "z_card": full["z_card"]}
            g = allreduce_f2_inputs(loc, dist, natural_x=True)
            t_sh, _ = d3.f2_decide(g["mx_hist"], g["mz_hist"], g["x_card"], g["y_card"],
                                   g["z_card"], g["out_j"], C)
            t_full, _ = d3.f2_decide(full["mx_hist"], full["mz_hist"], full["x_card"],
                                     full["y_card"], full["z_card"], full["out_j"], C)
            same_table = (g["out_j"] == full["out_j"] and np.array_equal(t_sh, t_full))
            # per-shard distinct pairs (brute force on the shard's R rows)
            keep = (r[0] >= lo) & (r[0] < hi)
            pairs = oracle_pairs((r[0][keep], r[1][keep]), s)
            xs = np.array([p[0] for p in pairs], np.uint64)
            zs = np.array([p[1] for p in pairs], np.uint64)
            n, x, sm = O.set_fingerprint(xs, zs) if len(pairs) else (0, 0, 0)
            tot = reduce_tally(n, sm, x, dist)
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
