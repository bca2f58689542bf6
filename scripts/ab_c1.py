"""A/B aid: configs[0] (GF(65521) u32, n = 10^5) per-launch time under the shipped tuning table vs the built-in
plan, CUDA-graph replay over rotating input copies (>= 3x L2), interleaved rounds."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp  # noqa: E402
import synth  # noqa: E402

p, n = 65521, 100_000
reps = [(torch.from_numpy(synth.uniform(synth.BASE_SEED, 0, 0, n, p, np.uint32)).cuda(),
         torch.from_numpy(synth.uniform(synth.BASE_SEED, 1, 0, n, p, np.uint32)).cuda()) for _ in range(480)]
out = torch.empty(1, dtype=torch.uint32, device="cuda")
s = torch.cuda.Stream()
ship = gfp.tune_entries()


def timed(label):
    with torch.cuda.stream(s):
        for a, b in reps[:4]:
            gfp.dot(a, b, p, out=out, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for a, b in reps:
                gfp.dot(a, b, p, out=out, stream=s)
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(5):
            g.replay()
        e1.record(s)
        s.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * len(reps))


for r in range(4):
    gfp.tune_set(ship)
    t_ship = timed("ship")
    kern_ship = gfp.plan(p, gfp.CLASSICAL, n, dtype=torch.uint32)["kernel"]
    gfp.tune_clear()
    t_bi = timed("builtin")
    kern_bi = gfp.plan(p, gfp.CLASSICAL, n, dtype=torch.uint32)["kernel"]
    print(f"round {r}: shipped table {t_ship:.3f} us ({kern_ship})   built-in {t_bi:.3f} us ({kern_bi})")
