"""Generates tests/golden/golden.json from the UNMODIFIED reference
(oracle/_ref/libdim3ref.so, built from /root/reference by oracle/Makefile).
Run here, where /root/reference exists; the JSON travels with the repo.

For each BASELINE config (convention G, test_consts()):
  * pipeline facts via the reference API (map_tables, build_csr,
    compute_degree_stats, partition_s_csr): cards, nnz, exact OUT_J, the
    dense/sparse z split and an order-independent fingerprint of the dense
    z set (count, xor and sum of mix64(z));
  * the full distinct (x, z) set fingerprint (count, sum, xor of
    mix64(mix64(x) ^ z)) via the reference sparse_bmm over row slices;
  * for cfg1/cfg2 the reference hybrid run's report (DenseEC counters,
    phase times on this container) — the W_D numerator of SURVEY 8(d);
  * cfg5: the x < 1000 slice of R against full S (the engine swaps), with
    per-block fingerprints keyed by raw x / 100.

Usage: python tests/golden/make_golden.py [cfg ...]   (default 1 2 3 4 5 55;
55 = the cfg5 100-x blocks spread over the whole x range)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
THREADS = os.cpu_count() or 8


def zfp(z):
    z = np.asarray(z, dtype=np.uint64)
    h = O.pair_hash_np(z, np.zeros_like(z))  # mix64(mix64(z) ^ 0)
    return {"count": int(z.size), "xor": int(np.bitwise_xor.reduce(h)) if z.size else 0,
            "sum": int(h.sum(dtype=np.uint64)) if z.size else 0}


def cfg5_block_ids():
    """100-x blocks spread over the whole cfg5 x range [0, 1e7): 20 evenly
    spaced (the first and the LAST block included) plus 4 seeded picks."""
    n_blocks = 10_000_000 // 100
    ids = {i * (n_blocks - 1) // 19 for i in range(20)}
    rng = np.random.default_rng(55)
    ids |= set(int(v) for v in rng.integers(0, n_blocks, 4))
    return sorted(ids)


def cfg5_blocks(data):
    """cfg5 per-block fingerprints over the whole x range. R restricted to the
    rows whose x falls in one of the blocks, against the full 200M-row S, run
    through the reference (its engine swaps, engine.cpp:361-366), with pairs
    bucketed by raw x / 100."""
    t0 = time.time()
    ids = cfg5_block_ids()
    r = O.gen(5, 0)
    s = O.gen(5, 1)
    blk = r.left // 100
    keep = np.isin(blk, np.asarray(ids, dtype=np.uint64))
    r = O.Table(np.ascontiguousarray(r.left[keep]), np.ascontiguousarray(r.right[keep]))
    n_blocks = 10_000_000 // 100
    cs = O.ref_set_checksum(r, s, threads=THREADS, rows_per_slice=65536,
                            block_width=100, n_blocks=n_blocks)
    entry = {"rows_r": len(r), "rows_s": len(s), "width": 100, "blocks": ids,
             "count": [int(cs["blk_count"][b]) for b in ids],
             "sum": [int(cs["blk_sum"][b]) for b in ids],
             "xor": [int(cs["blk_xor"][b]) for b in ids],
             "set": {k: cs[k] for k in ("count", "sum", "xor")},
             "seconds_to_generate": round(time.time() - t0, 1)}
    assert sum(entry["count"]) == cs["count"]
    data["cfg5_blocks"] = entry
    json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
    print("cfg5_blocks", len(ids), "blocks", json.dumps(entry["set"]),
          f"{time.time() - t0:.1f}s", flush=True)


def main(cfgs):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for cfg in cfgs:
        t0 = time.time()
        if cfg == 55:  # the cfg5 blocks over the whole x range
            cfg5_blocks(data)
            continue
        key = f"cfg{cfg}"
        r = O.gen(cfg, 0)
        s = O.gen(cfg, 1)
        entry = {"rows": len(r)}
        if cfg == 5:
            keep = r.left < 1000
            r = O.Table(np.ascontiguousarray(r.left[keep]), np.ascontiguousarray(r.right[keep]))
            key = "cfg5_x_lt_1000"
            entry = {"rows_r": len(r), "rows_s": len(s)}
            cs = O.ref_set_checksum(r, s, threads=THREADS, rows_per_slice=65536,
                                    block_width=100, n_blocks=10)
            entry["set"] = {k: cs[k] for k in ("count", "sum", "xor")}
            entry["blocks"] = {"width": 100, "count": cs["blk_count"].tolist(),
                               "sum": cs["blk_sum"].tolist(), "xor": cs["blk_xor"].tolist()}
        else:
            p = O.ref_pipeline(r, s)
            dz = p.pop("dense_z_raw")
            entry["pipeline"] = p
            entry["dense_z_fp"] = zfp(dz)
            rows_per_slice = {1: 1024, 2: 4096, 3: 1 << 18, 4: 8192}[cfg]
            cs = O.ref_set_checksum(r, s, threads=THREADS, rows_per_slice=rows_per_slice)
            entry["set"] = cs
            if cfg in (1, 2):
                rep = O.ref_join_project(r, s, force="hybrid", threads=THREADS, count_only=True,
                                         budget_bytes=1 << 40)
                entry["ref_hybrid_report"] = rep
        entry["seconds_to_generate"] = round(time.time() - t0, 1)
        data[key] = entry
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
        print(key, json.dumps(entry.get("set")), f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5, 55])
