"""A/B aid: the end-to-end headline leg -- gfp_dot_host of configs[2] (2 x 2^28 u32 Montgomery forms from pinned
host memory: chunked H2D overlapped with the dot kernels, result read back) -- per call and as GB/s of H2D."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp  # noqa: E402
import synth  # noqa: E402

p, n = 2 ** 31 - 1, 1 << 28
a = torch.from_numpy(synth.uniform(synth.BASE_SEED + 2, 0, 0, n, p, np.uint32)).pin_memory()
b = torch.from_numpy(synth.uniform(synth.BASE_SEED + 2, 1, 0, n, p, np.uint32)).pin_memory()
r0 = gfp.dot_host(a, b, p, gfp.MONTGOMERY)
ts = []
for _ in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = gfp.dot_host(a, b, p, gfp.MONTGOMERY)
    ts.append(time.perf_counter() - t0)
    assert r == r0
t = sorted(ts)[len(ts) // 2]
print(f"gfp_dot_host 2 x 2^28 u32: median {t * 1e3:.2f} ms, {2 * n * 4 / t / 1e9:.2f} GB/s H2D, {n / t:.3e} terms/s")
