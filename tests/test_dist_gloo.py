"""Multi-rank host logic of paper_cs_0404008_b200.dist on CPU: world_size 2 over gloo (127.0.0.1).

The device kernels are exercised by the GPU tests (virtual shards on one GPU); here the per-rank partial
residues come from the oracle (test-only stand-in), and what is checked is the layer's own logic:
the shard ranges, the int64 all_reduce of partials, and the row-block gather of the batch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

gfp_dist = pytest.importorskip("paper_cs_0404008_b200.dist")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        results = {}
        # ---- single dots: classical and Montgomery (the representation is linear in the partials)
        for p, rep, n in [(65521, 0, 100_003), (2 ** 31 - 1, 1, 77_777), (4294967291, 0, 5)]:
            a = synth.uniform(synth.BASE_SEED, 0, 0, n, p, np.uint32)
            b = synth.uniform(synth.BASE_SEED, 1, 0, n, p, np.uint32)
            s0, s1 = gfp_dist.shard_range(n, rank, world)
            if rep == 1:
                part = oracle.to_mont(p, oracle.dot_classical(p, a[s0:s1], b[s0:s1]))
            else:
                part = oracle.dot_classical(p, a[s0:s1], b[s0:s1])
            t = torch.tensor([part], dtype=torch.int64)
            gfp_dist.combine_partials(t)
            results[(p, rep)] = int(t.item()) % p  # what gfp_finalize computes before encoding
        # ---- batch rows with gather (stand-in row kernel from the oracle)
        p, rows, n = 65521, 37, 50
        A = synth.uniform(synth.BASE_SEED, 2, 0, rows * n, p, np.uint16).reshape(rows, n)
        x = synth.uniform(synth.BASE_SEED, 3, 0, n, p, np.uint16)
        r0, r1 = gfp_dist.shard_range(rows, rank, world)
        gfp_dist._dot_batch = lambda Ab, xb, p_, rep_, stream=None: torch.from_numpy(
            oracle.dot_batch_classical(p_, Ab.numpy(), xb.numpy()).astype(np.int64)).to(torch.int32)
        full = gfp_dist.dot_batch(torch.from_numpy(A[r0:r1]), torch.from_numpy(x), p, 0, gather=True)
        results["batch"] = full.to(torch.int64).tolist()
        q.put((rank, results, None))
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, None, repr(e)))


def test_shard_range_partitions():
    for n in [0, 1, 7, 100_003, 1 << 28]:
        for world in [1, 2, 3, 8]:
            spans = [gfp_dist.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [s1 - s0 for s0, s1 in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        gfp_dist.shard_range(5, 2, 2)


def test_gloo_world2_partials_and_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, res, err in out:
        assert err is None, err
        for p, rep, n in [(65521, 0, 100_003), (2 ** 31 - 1, 1, 77_777), (4294967291, 0, 5)]:
            a = synth.uniform(synth.BASE_SEED, 0, 0, n, p, np.uint32)
            b = synth.uniform(synth.BASE_SEED, 1, 0, n, p, np.uint32)
            want = oracle.dot_classical(p, a, b)
            assert res[(p, rep)] == (oracle.to_mont(p, want) if rep == 1 else want)
        p, rows, n = 65521, 37, 50
        A = synth.uniform(synth.BASE_SEED, 2, 0, rows * n, p, np.uint16).reshape(rows, n)
        x = synth.uniform(synth.BASE_SEED, 3, 0, n, p, np.uint16)
        assert res["batch"] == oracle.dot_batch_classical(p, A, x).astype(np.int64).tolist()
