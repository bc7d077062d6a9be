"""Summarise an ncu report (``ncu -i X.ncu-rep --page raw --csv``) or a launch
list (``--metrics gpu__time_duration.sum --csv``) into markdown.

usage: python profiles/summarize_ncu.py raw  <raw.csv>
       python profiles/summarize_ncu.py list <launches.csv>
"""
import collections
import csv
import sys

RAW_KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
]


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(k) for k, _ in RAW_KEYS if k in hdr}
    kn = hdr.index("Kernel Name")
    print("| kernel | " + " | ".join(lbl for k, lbl in RAW_KEYS if k in idx) + " |")
    print("|---" * (1 + len(idx)) + "|")
    for r in rows[2:]:
        name = r[kn].split("(")[0].replace("void ", "")
        cells = []
        for k, _ in RAW_KEYS:
            if k in idx:
                u = units[idx[k]]
                cells.append(f"{r[idx[k]]} {u}".strip())
        print(f"| {name} | " + " | ".join(cells) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    seq = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                seq.append((d["Kernel Name"].split("(")[0].replace("void ", "")[:70],
                            float(d["Metric Value"])))
    # the last step: from the last launch of the step's first kernel (the
    # fused column-statistics pass) on; the bench's peak micro-benchmarks and
    # the input generator are not part of a step
    starts = [i for i, (k, _) in enumerate(seq) if "colstat" in k]
    half = seq[starts[-1]:] if starts else seq[len(seq) // 2:]
    half = [(k, v) for k, v in half if "peak_kernel" not in k and "gen_kernel" not in k]
    agg = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, v in half:
        agg[k] += v
        cnt[k] += 1
    tot = sum(agg.values())
    print(f"launches in the step: {len(half)}; summed kernel time {tot / 1e6:.3f} ms "
          "(ncu: serialised, cold-cache — compare shares, not absolutes)\n")
    print("| kernel | ms | share | launches |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {v / 1e6:.3f} | {100 * v / tot:.1f}% | {cnt[k]} |")


if __name__ == "__main__":
    {"raw": raw, "list": launches}[sys.argv[1]](sys.argv[2])
