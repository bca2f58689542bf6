"""A/B aid: the pure-Zech dot (F3, GFP_STRAT_ZECH_ADD) at configs[3]'s shape (GF(32749), n = 2^26, 10% zeros) per call,
CUDA-graph replay over two input copies (512 MiB > 3x L2 between reuses); checks the result against the integer Zech
dot of the same library build."""
import sys

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
with torch.cuda.stream(s):
    want = gfp.dot(copies[0][0], copies[0][1], p, gfp.ZECH, stream=s)
    got = gfp.dot_ex(copies[0][0], copies[0][1], p, gfp.ZECH, strategy=gfp.ZECH_ADD, stream=s)
    s.synchronize()
assert torch.equal(want.cpu(), got.cpu()), (want, got)
per_graph = 20
with torch.cuda.stream(s):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(per_graph):
            x, y = copies[i % 2]
            gfp.dot_ex(x, y, p, gfp.ZECH, strategy=gfp.ZECH_ADD, out=out, stream=s)
    g.replay()
    s.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s)
    for _ in range(5):
        g.replay()
    e1.record(s)
    s.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (5 * per_graph)
print(f"pure-Zech dot p={p} n=2^26: {us:.2f} us  {n * 4 / us / 1e3:.0f} GB/s  (result equals the integer Zech dot)")
