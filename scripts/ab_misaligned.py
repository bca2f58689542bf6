"""A/B aid: a dot whose operands are not co-aligned (b offset by one element from a's 16-byte phase: the realigned
vector path since round 2, the scalar path before) vs the aligned vector path, for u32 (2^28) and u16 (2^27), back-to-back launches."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp  # noqa: E402
import synth  # noqa: E402


def timed(f, reps=20):
    s = torch.cuda.current_stream()
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s)
    for _ in range(reps):
        f()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for p, dt, n in [(2 ** 31 - 1, np.uint32, 1 << 28), (65521, np.uint16, 1 << 27)]:
    a = torch.from_numpy(synth.uniform(1, 0, 0, n + 8, p, dt)).cuda()
    b = torch.from_numpy(synth.uniform(1, 1, 0, n + 8, p, dt)).cuda()
    al = timed(lambda: gfp.dot(a[:n], b[:n], p, gfp.CLASSICAL))
    mis = timed(lambda: gfp.dot(a[:n], b[1:n + 1], p, gfp.CLASSICAL))
    both = timed(lambda: gfp.dot(a[1:n + 1], b[1:n + 1], p, gfp.CLASSICAL))
    nb = 2 * n * a.element_size()
    print(f"{np.dtype(dt).name} n={n}: aligned {al:.1f} us ({nb / al / 1e3:.0f} GB/s), a and b both +1 {both:.1f} us, "
          f"b alone +1 (not co-aligned) {mis:.1f} us ({nb / mis / 1e3:.0f} GB/s); kernel {gfp.plan(p, 0, n, dtype=torch.from_numpy(np.zeros(1, dt)).dtype)['kernel']}")
