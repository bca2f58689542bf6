"""Install-time tuning of the accumulation strategy (paper conclusion P:527-537).

    python -m paper_cs_0404008_b200.autotune [--out gfp_tune.txt] [--quick] [--ms 20]

Runs gfp_tune over a grid of (representation, prime, vector size) cases on cuda:0 -- the paper's
"determine and choose the best switching thresholds at install time" -- writes the table (load it with
gfp.tune_load(path) or export GFP_TUNE_FILE=path), and prints one JSON line per case with the winner and
its speed-up over the built-in plan.  Argument marshalling only: the measurements run in libgfp.
"""
from __future__ import annotations

import argparse
import json

import torch

import paper_cs_0404008_b200 as gfp

# primes: the paper's landmarks and the representation bounds (sec. 2), the switching points of sec. 3
U16_PRIMES = [3, 257, 2897, 2903, 16381, 32749, 46337, 65521]
# (65521 in u32 storage: configs[0]'s own case, a u16-size prime stored in 32-bit words)
U32_PRIMES = [65521, 65537, 1048573, 16777213, 268435399, 2 ** 31 - 1, 3037000493, 4294967291]
MONT_PRIMES = [40499, 65521, 2 ** 31 - 1, 2654435761]
FP_PRIMES = [32749, 65521, 67108859, 94906249]
ZECH_PRIMES = [32749, 65521]


def default_cases(quick: bool = False) -> list:
    ns = [1 << 12, 1 << 20] if quick else [1 << 12, 1 << 16, 1 << 20, 1 << 24]
    batches = [(1 << 14, 512)] if quick else [(1 << 15, 512), (1 << 12, 4096), (1 << 16, 4096)]
    cases = []

    def add(rep, primes, dtype=None, batch=True):
        for p in (primes[::3] + primes[-1:] if quick else primes):
            for n in ns:
                cases.append(dict(rep=rep, p=p, n=n, dtype=dtype))
            if batch:
                for rows, n in batches:
                    cases.append(dict(rep=rep, p=p, n=n, rows=rows, kind="batch", dtype=dtype))
    add(gfp.CLASSICAL, U16_PRIMES, torch.uint16)
    add(gfp.CLASSICAL, U32_PRIMES, torch.uint32)
    add(gfp.MONTGOMERY, MONT_PRIMES)
    add(gfp.FP64, FP_PRIMES)
    add(gfp.ZECH, ZECH_PRIMES)
    return cases


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--out", default="gfp_tune.txt")
    ap.add_argument("--quick", action="store_true", help="a small grid (CI / smoke)")
    ap.add_argument("--ms", type=float, default=20.0, help="milliseconds of timing per candidate")
    ap.add_argument("--min-gain", type=float, default=1.05,
                    help="keep a tuned strategy only if it beats the built-in plan by this factor; below it the "
                         "entry records AUTO, so run-to-run noise at the tuning sizes does not switch kernels")
    args = ap.parse_args(argv)
    torch.cuda.set_device(0)
    gfp.tune_clear()
    table = gfp.tune(default_cases(args.quick), ms_per_candidate=args.ms)
    for e in table:
        e["speedup_vs_builtin"] = e["us_builtin"] / e["us_best"] if e["us_best"] > 0 else None
        e["measured_winner"] = e["strategy_name"]
        if e["strategy"] != gfp.AUTO and (e["speedup_vs_builtin"] or 0) < args.min_gain:
            e.update(strategy=gfp.AUTO, acc_bits=0, us_best=e["us_builtin"], strategy_name="auto")
    gfp.tune_set(table)
    gfp.tune_save(args.out)
    for e in table:
        print(json.dumps(e), flush=True)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
