#!/usr/bin/env python
"""Render a bench.py --sweep JSONL file as a text table (terms/s in units of 10^12 per strategy), plus the
cost of one reduction per row fitted from the one-lane blocked32 column."""
import collections
import json
import sys

import numpy as np

cells = [json.loads(line) for line in open(sys.argv[1])]
by = collections.defaultdict(dict)
for c in cells:
    by[c["p"]][c["strategy"]] = c
names = ["auto", "builtin", "blocked32", "hybrid32", "blocked32_1lane", "hybrid32_1lane", "delayed64_1lane",
         "overflow32", "carry32", "blocked64", "overflow64", "hybrid64", "carry64"]
short = {"blocked32_1lane": "blk32_1L", "hybrid32_1lane": "hyb32_1L", "delayed64_1lane": "del64_1L"}
print("# F1 prime sweep (bench.py --sweep): DIM=512 dots, %d rows per cell; terms/s / 1e12 per strategy" % cells[0].get("rows", 0)
      if "rows" in cells[0] else "# F1 prime sweep (bench.py --sweep): DIM=512 dots; terms/s / 1e12 per strategy")
print("# auto = AUTO with the shipped install-time table, builtin = AUTO without it; columns without _1L run the "
      "library's 8 lanes per row (64 terms per accumulator), _1L one accumulator per row (the paper's loop, 512 terms)")
print("# k32 = blocked block length at m=32; red/row1L = reductions per row with one lane (ceil(512/k32)); "
      "red/lane8 = reductions per accumulator with 8 lanes (ceil(64/k32))")
print("# all cells bit-equal to the default plan: %s" % all(c["equal_to_default"] for c in cells))
print("p".rjust(11), *[short.get(n, n).rjust(10) for n in names], "k32".rjust(11), "red/row1L".rjust(10),
      "red/lane8".rjust(10))
for p in sorted(by):
    row = [f"{by[p][n]['terms_per_s'] / 1e12:10.3f}" if n in by[p] else " " * 10 for n in names]
    b = by[p].get("blocked32", {})
    b1 = by[p].get("blocked32_1lane", {})
    print(str(p).rjust(11), *row, str(b.get("block_k", "")).rjust(11), str(b1.get("reductions_per_lane", "")).rjust(10),
          str(b.get("reductions_per_lane", "")).rjust(10))

# cost of one reduction per accumulator, least squares over the primes: time per launch = t0 + c * reductions;
# and the two steps side by side -- the paper's (one lane, 2897 -> 2903) and the 8-lane kernel's (8191 -> 8209)
def fit(strategy):
    pts = [(c["reductions_per_lane"], c["us"]) for c in cells if c["strategy"] == strategy and c["reductions_per_lane"]]
    if len(pts) < 4:
        return None
    r = np.array([x for x, _ in pts], float)
    t = np.array([y for _, y in pts], float)
    (t0, cost), *_ = np.linalg.lstsq(np.stack([np.ones_like(r), r], 1), t, rcond=None)
    return t0, cost, len(pts)


def step(strategy, lo, hi):
    a, b = by.get(lo, {}).get(strategy), by.get(hi, {}).get(strategy)
    if not (a and b):
        return
    d = b["us"] - a["us"]
    sep = b.get("us_min", b["us"]) > a.get("us_max", a["us"])
    print("#   %s %d -> %d: reductions per accumulator %s -> %s; median %.3f -> %.3f us (%+.2f%%); replay ranges "
          "[%.3f, %.3f] / [%.3f, %.3f]%s" % (strategy, lo, hi, a["reductions_per_lane"], b["reductions_per_lane"],
                                             a["us"], b["us"], 100 * d / a["us"], a.get("us_min", a["us"]),
                                             a.get("us_max", a["us"]), b.get("us_min", b["us"]), b.get("us_max", b["us"]),
                                             " -- separated" if sep else " -- overlapping"))


print()
for strat in ("blocked32_1lane", "blocked32"):
    f = fit(strat)
    if f:
        t0, cost, k = f
        print("# %s: time per launch = %.3f us + %.4f us x (reductions per accumulator)   [least squares, %d primes]"
              % (strat, t0, cost, k))
step("blocked32_1lane", 2887, 2897)
step("blocked32_1lane", 2897, 2903)
step("hybrid32_1lane", 2897, 2903)
step("blocked32", 2897, 2903)
step("blocked32", 8191, 8209)
