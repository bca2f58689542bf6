"""A/B aid: configs[2] (GF(2^31-1) Montgomery dot, n = 2^28) per launch, back-to-back launches as bench.py times
them, for the Montgomery accumulation strategies: REDC every k_R = 2 products (the built-in plan), the carry word
(MontgomeryCarry: products summed with the carry flag counted, one REDC per thread), overflow-Montgomery."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp  # noqa: E402
import synth  # noqa: E402

p, n = 2 ** 31 - 1, 1 << 28
a = gfp.to_rep(torch.from_numpy(synth.uniform(synth.BASE_SEED + 2, 0, 0, n, p, np.uint32)).cuda(), p, gfp.MONTGOMERY)
b = gfp.to_rep(torch.from_numpy(synth.uniform(synth.BASE_SEED + 2, 1, 0, n, p, np.uint32)).cuda(), p, gfp.MONTGOMERY)
out = torch.empty(1, dtype=torch.uint32, device="cuda")
s = torch.cuda.Stream()
variants = {"builtin (REDC every 2)": lambda: gfp.dot(a, b, p, gfp.MONTGOMERY, out=out, stream=s),
            "carry word": lambda: gfp.dot_ex(a, b, p, gfp.MONTGOMERY, strategy=gfp.CARRY, out=out, stream=s),
            "overflow": lambda: gfp.dot_ex(a, b, p, gfp.MONTGOMERY, strategy=gfp.OVERFLOW, out=out, stream=s)}
ref = None
for name, f in variants.items():
    with torch.cuda.stream(s):
        f()
    s.synchronize()
    v = int(out.cpu().to(torch.int64)[0])
    ref = v if ref is None else ref
    assert v == ref, name
for rnd in range(3):
    for name, f in variants.items():
        with torch.cuda.stream(s):
            for _ in range(5):
                f()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s)
            for _ in range(100):
                f()
            e1.record(s)
        s.synchronize()
        us = e0.elapsed_time(e1) * 10
        print(f"round {rnd} {name:24s} {us:7.1f} us per launch  {2 * n * 4 / us / 1e3:.0f} GB/s")
