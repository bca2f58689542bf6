import torch, numpy as np, paper_cs_0404008_b200 as g, synth
for p in [32749, 32771, 40009, 65521]:
    for n in [0, 1, 4096, 100003]:
        a = torch.from_numpy(synth.zech_codes(1, 0, 0, n, p - 1)).cuda()
        b = torch.from_numpy(synth.zech_codes(1, 1, 0, n, p - 1)).cuda()
        try:
            r = g.dot_ex(a, b, p, g.ZECH, strategy=g.ZECH_ADD); torch.cuda.synchronize()
            print(p, n, 'ok', g.plan(p, g.ZECH, n, strategy=g.ZECH_ADD)['grid'])
        except Exception as e:
            print(p, n, 'ERR', e, g.plan(p, g.ZECH, n, strategy=g.ZECH_ADD))
