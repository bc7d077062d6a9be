#!/usr/bin/env python
"""Kernel launch list of ONE rank of an N-rank sharded join_project (the
shard projection's method, scripts/shard_projection.py): the N ranks run as
threads with a recorded exchange, then rank --rank is replayed alone between
cudaProfilerStart/Stop, so

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \\
      python scripts/shard_trace.py --config 5 --shards 8 --rank 0

lists that rank's kernels only. Prints the replayed call's phase times."""
import argparse
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    a = ap.parse_args()
    import torch

    import paper_2206_04995_b200 as d3
    from paper_2206_04995_b200.distributed import (RecordingExchange, ReplayExchange,
                                                   ThreadExchange)
    x_card = {1: 10_000, 2: 200_000, 3: 2_000_000, 5: 10_000_000}[a.config]
    C = d3.CostConstants.test_consts()
    rl, rr = d3.generate(a.config, 0)
    sl, sr = d3.generate(a.config, 1)
    S = d3.RawTable(sl, sr)
    e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True,
                        memory_budget_bytes=150 << 30)
    n = a.shards
    shards = []
    for q in range(n):
        lo, hi = x_card * q // n, x_card * (q + 1) // n
        m = (rl >= lo) & (rl < hi)
        shards.append(d3.RawTable(rl[m].contiguous(), rr[m].contiguous()))
    ctxs = [d3.Context(0) for _ in range(n)]
    te = ThreadExchange(n)
    recs = [RecordingExchange(te.rank_fn(q)) for q in range(n)]

    def rank_main(q):
        ctxs[q].set_exchange(n, q, recs[q])
        d3.join_project(shards[q], S, e, C, ctx=ctxs[q])

    th = [threading.Thread(target=rank_main, args=(q,)) for q in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    q = a.rank
    for c in range(n):
        if c != q:
            ctxs[c].close()
    rp = ReplayExchange(list(recs[q].log))
    ctxs[q].set_exchange(n, q, rp)
    d3.join_project(shards[q], S, e, C, ctx=ctxs[q])  # warm (pool, modules)
    rp.rewind()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    rep = d3.join_project(shards[q], S, e, C, ctx=ctxs[q]).report
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print({k: round(getattr(rep, k), 3) for k in
           ("ms_total", "ms_exchange_host", "ms_map", "ms_csr", "ms_stats", "ms_partition",
            "ms_dense", "ms_dense_hot", "ms_dense_cold")}, "zsplit", rep.zsplit,
          "bus_bytes", rep.exchange_bus_bytes, "calls", rep.exchange_calls)


if __name__ == "__main__":
    main()
