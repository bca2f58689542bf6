"""A/B aid: Zech conversions of configs[3]'s two operands (2 x 2^26 u16), per pair, CUDA-graph replay."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp  # noqa: E402
import synth  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.Stream()
p, n = 32749, 1 << 26
a = torch.from_numpy(synth.zech_codes(synth.BASE_SEED + 3, 0, 0, n, p - 1)).cuda()
b = torch.from_numpy(synth.zech_codes(synth.BASE_SEED + 3, 1, 0, n, p - 1)).cuda()
ra, rb = torch.empty_like(a), torch.empty_like(b)
ca, cb = torch.empty_like(a), torch.empty_like(b)
for name, f in [("from_zech", lambda: (gfp.from_rep(a, p, gfp.ZECH, out=ra, stream=s), gfp.from_rep(b, p, gfp.ZECH, out=rb, stream=s))),
                ("to_zech", lambda: (gfp.to_rep(ra, p, gfp.ZECH, out=ca, stream=s), gfp.to_rep(rb, p, gfp.ZECH, out=cb, stream=s)))]:
    with torch.cuda.stream(s):
        f()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(5):
                f()
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(4):
            g.replay()
        e1.record(s)
        s.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    print(f"{name}: {us:.1f} us per pair  {4 * 2 * n / us / 1e3:.0f} GB/s r+w")
assert torch.equal(ca, a) and torch.equal(cb, b)
