#!/usr/bin/env python
"""Render a bench.py --sweep JSONL file as a text table (terms/s in units of 10^12 per strategy)."""
import collections
import json
import sys

cells = [json.loads(line) for line in open(sys.argv[1])]
by = collections.defaultdict(dict)
for c in cells:
    by[c["p"]][c["strategy"]] = c
names = ["auto", "builtin", "blocked32", "overflow32", "hybrid32", "carry32", "blocked64", "overflow64", "hybrid64", "carry64"]
print("# F1 prime sweep (bench.py --sweep): DIM=512 dots, 2^19 rows per cell; terms/s / 1e12 per strategy (auto = AUTO with the shipped install-time table, builtin = AUTO without it); k32 = blocked "
      "block length at m=32; red/lane32 = reductions per lane (16 terms); all cells bit-equal to the default plan: %s"
      % all(c["equal_to_default"] for c in cells))
print("p".rjust(11), *[n.rjust(10) for n in names], "k32".rjust(11), "red/lane32".rjust(10))
for p in sorted(by):
    row = [f"{by[p][n]['terms_per_s'] / 1e12:10.2f}" if n in by[p] else " " * 10 for n in names]
    b = by[p].get("blocked32", {})
    print(str(p).rjust(11), *row, str(b.get("block_k", "")).rjust(11), str(b.get("reductions_per_lane", "")).rjust(10))
