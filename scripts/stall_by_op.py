"""Aggregate an ncu source-page CSV (--page source --csv --print-source sass) by SASS opcode: warp-stall samples
per stall reason, so the binding dependency (global load, shared load, math chain) is visible at a glance.

    python scripts/stall_by_op.py gpurun_out/zs/src_default_32749.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[idx["Source"]].split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    for h in reasons:
        v = int(r[idx[h]] or 0)
        byop[o][h] += v
        tot[h] += v
allsum = sum(tot.values())
print("total samples", allsum)
for h, v in tot.most_common(10):
    print(f"  {h:28s} {v:8d} {100 * v / allsum:5.1f}%")
print("by opcode (samples, top reasons):")
for o, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    s = sum(c.values())
    print(f"  {o:10s} {s:8d} {100 * s / allsum:5.1f}%  " + ", ".join(f"{h[6:]}={v}" for h, v in c.most_common(4)))
