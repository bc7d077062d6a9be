"""Opcode histogram and hottest SASS lines of one kernel from
`ncu -i X.ncu-rep --page source --csv --kernel-name regex:K` (diagnostic)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if r and r[0] == "Address"][0]
idx = {n: i for i, n in enumerate(hdr)}
ie, sm, src = idx["Instructions Executed"], idx["# Samples"], idx["Source"]
data = [r for r in rows if len(r) == len(hdr) and r[ie].isdigit()]
tot = sum(int(r[ie]) for r in data)
samp = sum(int(r[sm]) for r in data)
print("total warp inst", tot, "samples", samp, "sass lines", len(data))
op, ops = collections.Counter(), collections.Counter()
for r in data:
    m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9_.]+)", r[src])
    o = m.group(2).split(".")[0] if m else "?"
    op[o] += int(r[ie])
    ops[o] += int(r[sm])
for o, c in op.most_common(20):
    print(f"{o:10s} {c / tot * 100:5.1f}% inst  {ops[o] / samp * 100:5.1f}% samples")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
top = sorted(range(len(data)), key=lambda i: -int(data[i][sm]))[:n]
for i in sorted(top):
    print(i, data[i][src].strip()[:70], data[i][ie], data[i][sm])
