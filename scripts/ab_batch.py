"""A/B timing of batch strategies (tuning aid, not the product): alternating order, rotating inputs."""
import sys
import torch
import numpy as np
sys.path.insert(0, ".")
import paper_cs_0404008_b200 as gfp
import synth

torch.cuda.set_device(0)
gfp.tune_clear()
dev = "cuda:0"
for p, dt, rows, n, rep in [(2 ** 31 - 1, np.uint32, 32768, 512, 0), (16777213, np.uint32, 32768, 512, 0),
                            (2 ** 31 - 1, np.uint32, 4096, 4096, 0), (2 ** 31 - 1, np.uint32, 32768, 512, 1),
                            (65521, np.float64, 4096, 4096, 2)]:
    sets = [torch.from_numpy(synth.uniform(k, 2, 0, rows * n, p, dt)).to(dev).view(rows, n) for k in range(8)]
    x = torch.from_numpy(synth.uniform(1, 3, 0, n, p, dt)).to(dev)
    cands = {"builtin": (gfp.AUTO, 0)}
    if rep == 0:
        cands.update({"hybrid64": (gfp.HYBRID, 64), "blocked64": (gfp.BLOCKED, 64), "carry64": (gfp.CARRY, 64)})
    elif rep == 1:
        cands.update({"carry": (gfp.CARRY, 0), "overflow": (gfp.OVERFLOW, 0)})
    else:
        cands.update({"blocked": (gfp.BLOCKED, 0), "delayed": (gfp.DELAYED, 0)})
    res = {k: [] for k in cands}
    for it in range(6):
        order = list(cands) if it % 2 == 0 else list(reversed(list(cands)))
        for k in order:
            s, m = cands[k]
            for w in range(3):
                gfp.dot_batch_ex(sets[w], x, p, rep, strategy=s, acc_bits=m)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for r in range(40):
                gfp.dot_batch_ex(sets[r % 8], x, p, rep, strategy=s, acc_bits=m)
            e1.record()
            torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 1e3 / 40)
    print(p, rep, rows, n, {k: round(min(v), 2) for k, v in res.items()},
          {k: gfp.plan(p, rep, n, dtype=sets[0].dtype, strategy=cands[k][0], acc_bits=cands[k][1])["kernel"] for k in cands})
