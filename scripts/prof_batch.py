"""One u32 batch launch for ncu (tuning aid)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp
import synth
import numpy as np
p, rows, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
strat = int(sys.argv[4]) if len(sys.argv) > 4 else 0
bits = int(sys.argv[5]) if len(sys.argv) > 5 else 0
A = torch.from_numpy(synth.uniform(1, 2, 0, rows * n, p, np.uint32)).cuda().view(rows, n)
x = torch.from_numpy(synth.uniform(1, 3, 0, n, p, np.uint32)).cuda()
for _ in range(3):
    gfp.dot_batch_ex(A, x, p, 0, strategy=strat, acc_bits=bits)
torch.cuda.synchronize()
