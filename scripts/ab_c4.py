"""A/B aid: configs[3] (GF(32749) Zech dot, n = 2^26, 10% zeros) per call, CUDA-graph replay over two input copies
(512 MiB > 3x L2 between reuses), plus a small-n call (2^16) for the per-launch fixed cost; checks the result."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp  # noqa: E402
import synth  # noqa: E402

p, n = 32749, 1 << 26
a = synth.zech_codes(synth.BASE_SEED + 3, 0, 0, n, p - 1)
b = synth.zech_codes(synth.BASE_SEED + 3, 1, 0, n, p - 1)
copies = [(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) for _ in range(2)]
out = torch.empty(1, dtype=torch.uint16, device="cuda")
s = torch.cuda.Stream()
print("kernel:", gfp.plan(p, gfp.ZECH, n)["kernel"])


def timed(pairs, per_graph):
    with torch.cuda.stream(s):
        for x, y in pairs[:2]:
            gfp.dot(x, y, p, gfp.ZECH, out=out, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(per_graph):
                x, y = pairs[i % len(pairs)]
                gfp.dot(x, y, p, gfp.ZECH, out=out, stream=s)
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(5):
            g.replay()
        e1.record(s)
        s.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * per_graph)


r = int(gfp.dot(copies[0][0], copies[0][1], p, gfp.ZECH).cpu().to(torch.int64)[0])
for _ in range(3):
    print(f"C4: {timed(copies, 16):.2f} us per call   result code {r}")
small = [(x[: 1 << 16], y[: 1 << 16]) for x, y in copies] * 64
print(f"n = 2^16: {timed(small, 128):.2f} us per call")
