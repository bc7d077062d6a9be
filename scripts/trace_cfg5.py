"""Phase times of one cfg5 call in a given mode (diagnostic; D3G_TRACE=1 adds
the DenseEC split). Usage: python scripts/trace_cfg5.py [count|checksum] [shard/of]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_04995_b200 as d3  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "count"
shard = (0, 1)
if len(sys.argv) > 2:
    a, b = sys.argv[2].split("/")
    shard = (int(a), int(b))
cfg = int(os.environ.get("CFG", "5"))
C = d3.CostConstants.test_consts()
rl, rr = d3.generate(cfg, 0)
sl, sr = d3.generate(cfg, 1)
e = d3.EngineConfig(force=d3.Strategy.auto_select, count_only=True, checksum=(mode == "checksum"),
                    memory_budget_bytes=120 << 30, shard_index=shard[0], shard_count=shard[1])
for i in range(2):
    t0 = time.perf_counter()
    rep = d3.join_project(d3.RawTable(rl, rr), d3.RawTable(sl, sr), e, C).report
    wall = time.perf_counter() - t0
print(f"{mode} shard {shard}: wall {wall*1e3:.1f} ms  out_p {rep.out_p}")
for k in ("ms_map", "ms_csr", "ms_stats", "ms_partition", "ms_sparse", "ms_dense", "ms_dense_hot",
          "ms_dense_cold", "ms_total", "hot_direct_pairs", "cold_bytes", "gpu_launches"):
    print(f"  {k} = {getattr(rep, k)}")
