"""One Zech matrix-vector launch (65536 x 4096 u16 codes) per prime given, after warm-up, for ncu."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp  # noqa: E402
import synth  # noqa: E402

rows, n = 65536, 4096
for p in [int(v) for v in sys.argv[1:]] or [32749]:
    A = torch.from_numpy(synth.zech_codes(5, 2, 0, rows * n, p - 1).reshape(rows, n)).cuda()
    x = torch.from_numpy(synth.zech_codes(5, 3, 0, n, p - 1)).cuda()
    for _ in range(3):
        gfp.dot_batch(A, x, p, gfp.ZECH)
    torch.cuda.synchronize()
    del A, x
