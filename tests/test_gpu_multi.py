"""Multi-GPU parity: one process per visible GPU (NCCL over NVLink), every BASELINE.json config sharded
across them, through BOTH combines of the multi-GPU layer -- `dist.dot` (gfp_dot_partial, one int64 NCCL
all_reduce, gfp_finalize) and `dist.dot_fused` (ONE kernel per rank whose last CTA exchanges the shard's
partial over peer memory and finalizes, gfp_dot_allreduce) -- and the row-sharded matrix-vector product
(`dist.dot_batch`, gather=True).  Every rank's result is compared with the oracle on the whole (unsharded)
input, computed once in the parent.

Needs >= 2 GPUs: it SKIPS on a one-GPU box (this round's gpurun boxes and the driver's round-end GPU tests
have one).  Ranks whose kernels wait on one another are never simulated on one GPU (B200_PROFILING.md);
the one-GPU evidence for the fused path is test_gpu_xchg_ipc.py and the protocol model.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

P31 = 2 ** 31 - 1
# (name, p, rep, kind, n or (rows, n)) -- BASELINE.json configs[0..4] at full size
CONFIGS = [("C1", 65521, 0, "dot", 100_000), ("C2", 67108859, 2, "dot", 10 ** 7),
           ("C3", P31, 1, "dot", 1 << 28), ("C4", 32749, 3, "dot", 1 << 26),
           ("C5", 65521, 0, "batch", (65536, 4096))]


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _inputs(i, name, p, rep, kind, size, lo=None, hi=None):
    """Host inputs of config i (elements / rows [lo, hi)), in the representation's INPUT form (classical
    residues for Montgomery, converted on the device)."""
    seed = synth.BASE_SEED + i
    if kind == "batch":
        rows, n = size
        lo, hi = (0, rows) if lo is None else (lo, hi)
        A = synth.uniform(seed, synth.STREAM_MAT, lo * n, (hi - lo) * n, p, np.uint16).reshape(hi - lo, n)
        return A, synth.uniform(seed, synth.STREAM_X, 0, n, p, np.uint16)
    lo, hi = (0, size) if lo is None else (lo, hi)
    if rep == 3:
        return (synth.zech_codes(seed, synth.STREAM_A, lo, hi - lo, p - 1),
                synth.zech_codes(seed, synth.STREAM_B, lo, hi - lo, p - 1))
    dt = np.float64 if rep == 2 else np.uint32
    return synth.uniform(seed, synth.STREAM_A, lo, hi - lo, p, dt), synth.uniform(seed, synth.STREAM_B, lo, hi - lo, p, dt)


def _expected():
    want = {}
    for i, (name, p, rep, kind, size) in enumerate(CONFIGS):
        a, b = _inputs(i, name, p, rep, kind, size)
        if kind == "batch":
            want[name] = oracle.dot_batch_classical(p, a, b).astype(np.int64).tolist()
        elif rep == 1:
            want[name] = oracle.to_mont(p, oracle.dot_classical(p, a, b))  # result in Montgomery form
        else:
            want[name] = oracle.dot(p, rep, a, b)
    return want


def _worker(rank, world, port, want, q):
    try:
        import torch.distributed as dist

        import paper_cs_0404008_b200 as gfp
        from paper_cs_0404008_b200 import dist as gdist
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                                device_id=dev)
        xchg = gdist.PeerExchange()
        bad = []
        for i, (name, p, rep, kind, size) in enumerate(CONFIGS):
            if kind == "batch":
                r0, r1 = gdist.shard_range(size[0], rank, world)
                A, x = _inputs(i, name, p, rep, kind, size, r0, r1)
                got = gdist.dot_batch(torch.from_numpy(A).to(dev), torch.from_numpy(x).to(dev), p, rep, gather=True)
                if got.cpu().to(torch.int64).tolist() != want[name]:
                    bad.append((name, "batch"))
                continue
            s0, s1 = gdist.shard_range(size, rank, world)
            a, b = _inputs(i, name, p, rep, kind, size, s0, s1)
            a, b = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
            if rep == 1:
                a, b = gfp.to_rep(a, p, rep), gfp.to_rep(b, p, rep)
            for how, f in (("nccl", lambda: gdist.dot(a, b, p, rep)),
                           ("fused", lambda: gdist.dot_fused(a, b, p, rep, xchg))):
                for _ in range(3):  # repeated epochs (both slot parities of the fused exchange)
                    r = f().cpu()
                    v = r[0].item() if r.dtype == torch.float64 else int(r.to(torch.int64)[0])
                    if v != want[name]:
                        bad.append((name, how, v, want[name]))
        torch.cuda.synchronize()
        xchg.close()
        dist.destroy_process_group()
        q.put((rank, bad, None))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, None, repr(e)))


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (one process per GPU); this box has fewer")
def test_multi_gpu_configs_both_combines():
    import torch.multiprocessing as mp
    world = min(_ngpus(), 8)
    want = _expected()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, want, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=900) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
    for rank, bad, err in out:
        assert err is None, (rank, err)
        assert bad == [], (rank, bad)
