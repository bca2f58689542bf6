"""Per-call latency of small dots in CUDA-graph replay (tuning aid): Zech (table staging) vs classical."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp
import synth

torch.cuda.set_device(0)
s = torch.cuda.Stream()
for name, p, rep, dt, n in [("classical u16", 65521, gfp.CLASSICAL, np.uint16, 1 << 16),
                            ("zech 32749", 32749, gfp.ZECH, np.uint16, 1 << 16),
                            ("zech 65521 (large)", 65521, gfp.ZECH, np.uint16, 1 << 16),
                            ("zech_add 32749", 32749, -5, np.uint16, 1 << 16),
                            ("fp64", 67108859, gfp.FP64, np.float64, 1 << 16),
                            ("classical u32 1e5", 65521, gfp.CLASSICAL, np.uint32, 100000)]:
    if rep in (gfp.ZECH, -5):
        a = torch.from_numpy(synth.zech_codes(1, 0, 0, n, p - 1)).cuda()
    else:
        a = torch.from_numpy(synth.uniform(1, 0, 0, n, p, dt)).cuda()
    out = torch.empty(1, dtype=a.dtype, device="cuda")
    call = (lambda: gfp.dot_ex(a, a, p, gfp.ZECH, strategy=gfp.ZECH_ADD, out=out, stream=s)) if rep == -5 else \
        (lambda: gfp.dot(a, a, p, rep, out=out, stream=s))
    with torch.cuda.stream(s):
        call()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                call()
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(10):
            g.replay()
        e1.record(s)
        s.synchronize()
    print(f"{name:24s} n={n:7d}  {e0.elapsed_time(e1) * 1e3 / 500:.2f} us/call")
