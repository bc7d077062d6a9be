"""Extra randomized parity run on a B200 (not part of the suite): 160 random
instances (a third of them larger: up to 60k rows over 4096-value domains) x 4
strategies x {default, forced hash cold pass, hash pass with tiny tier limits}, materialized set and count-only
count against the brute-force oracle. python scripts/stress_extra.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2206_04995_b200 as d3
from support import SplitMix64, random_instance, oracle_pairs, pair_set
C = d3.CostConstants.test_consts()
bad = 0; n = 0
for seed in (9001, 9002, 9003, 9004):
    rng = SplitMix64(seed)
    for it in range(40):
        if it % 3 == 0:
            r, s = random_instance(rng, 4096, 60000, 3000000)
        else:
            r, s = random_instance(rng)
        want = oracle_pairs(r, s)
        for f in (d3.Strategy.auto_select, d3.Strategy.hybrid, d3.Strategy.dense_only, d3.Strategy.sparse_only):
            for env in ({}, {"D3G_COLD_PATH": "hash"},
                        # tiny tier limits: the warp tier hands on to the CTA tier and that to the bitmap tier
                        {"D3G_COLD_PATH": "hash", "D3G_COLD_HASH_MAX": "32", "D3G_COLD_CTA_MAX": "64",
                         "D3G_COLD_STAR": "8"}):
                for k, v in env.items(): os.environ[k] = v
                out = d3.join_project(d3.RawTable(*r), d3.RawTable(*s), d3.EngineConfig(force=f), C)
                cnt = d3.join_project(d3.RawTable(*r), d3.RawTable(*s), d3.EngineConfig(force=f, count_only=True), C)
                for k in env: del os.environ[k]
                n += 1
                if pair_set(out.result.raw_x, out.result.raw_z) != want or cnt.report.out_p != len(want):
                    bad += 1
                    print("MISMATCH", seed, it, f, env, out.report.out_p, cnt.report.out_p, len(want))
print("runs", n, "bad", bad)
