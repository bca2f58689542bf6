"""A/B aid: Zech batch (65536 x 4096 u16 codes, GF(32749) and GF(65521)) per-call time, CUDA-graph replay."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp
import synth

torch.cuda.set_device(0)
s = torch.cuda.Stream()
for p in (32749, 65521):
    rows, n = 65536, 4096
    A = torch.from_numpy(synth.zech_codes(5, 2, 0, rows * n, p - 1).reshape(rows, n)).cuda()
    x = torch.from_numpy(synth.zech_codes(5, 3, 0, n, p - 1)).cuda()
    out = torch.empty(rows, dtype=torch.uint16, device="cuda")
    with torch.cuda.stream(s):
        gfp.dot_batch(A, x, p, gfp.ZECH, out=out, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                gfp.dot_batch(A, x, p, gfp.ZECH, out=out, stream=s)
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(5):
            g.replay()
        e1.record(s)
        s.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 50
    print(f"zech batch p={p}: {us:.1f} us  {rows * n * 2 / us / 1e3:.0f} GB/s")
