"""The fused multi-GPU combine (gfp_dot_allreduce) across two PROCESSES on one GPU, with real CUDA-IPC
exchange buffers -- without ranks whose kernels wait on one another.

Only rank 0 runs the fused kernel (world = 2).  Rank 1 plays its peer from the host: before each of rank
0's launches it publishes its tagged partial (epoch << 32 | residue) into rank 0's buffer through its own
IPC mapping; after the launch it reads its own buffer and checks that rank 0's kernel delivered rank 0's
tagged partial there (a system-scope store into another process's memory).  Rank 0 checks the encoded
result against the oracle: (partial_0 + partial_1) mod p in the representation.  So the whole data path
of the fused combine -- handle exchange, gfp_xchg_open in another process, the kernel's peer stores, the
tag polling, the parity slots over several epochs -- runs for real; what one GPU cannot show is two
kernels spinning on each other, which the protocol model (test_xchg_protocol.py) covers.

The exchange-buffer layout (word offsets) mirrors paper_cs_0404008_b200/csrc/internal.h.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

MAXW = 16
K_SLOTS = 8 + 2 * MAXW  # internal.h: kXSlots (tagged slots: epoch << 32 | residue)
K_WORDS = 8 + 5 * MAXW


class _Raw:
    """A device pointer as an int64 tensor (no copy) via __cuda_array_interface__."""

    def __init__(self, ptr, words):
        self.__cuda_array_interface__ = {"shape": (words,), "typestr": "<i8", "data": (ptr, False), "version": 3}


def _words(ptr):
    return torch.as_tensor(_Raw(ptr, K_WORDS), device="cuda:0")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# (p, rep, dtype, generator) for the epochs; the partials are in the representation's additive form
CASES = [(65521, 0, np.uint32, "u"), (2 ** 31 - 1, 1, np.uint32, "u"), (67108859, 2, np.float64, "u"),
         (32749, 3, np.uint16, "z"), (65521, 0, np.uint32, "u"), (2 ** 31 - 1, 1, np.uint32, "u")]


def _shard(rank, p, gen, dt, n):
    seed = synth.BASE_SEED + 17 * rank
    if gen == "z":
        return synth.zech_codes(seed, 0, 0, n, p - 1), synth.zech_codes(seed, 1, 0, n, p - 1)
    return synth.uniform(seed, 0, 0, n, p, dt), synth.uniform(seed, 1, 0, n, p, dt)


def _additive_partial(p, rep, a, b):
    """The shard's partial in the form the kernels exchange: classical residue (Montgomery: its form)."""
    if rep == 1:
        return oracle.dot_montgomery(p, a, b)
    if rep == 3:
        return oracle.zech_decode(p, 2, oracle.dot_zech(p, 2, a, b))
    return int(oracle.dot(p, rep, a, b))


def _worker(rank, port, q):
    try:
        import torch.distributed as dist
        import paper_cs_0404008_b200 as gfp
        from paper_cs_0404008_b200 import dist as gd
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
        x = gd.PeerExchange()
        assert x.world == 2 and x.rank == rank
        mine, peer = _words(x.ptrs[rank]), _words(x.ptrs[1 - rank])
        n = 300_007
        for e, (p, rep, dt, gen) in enumerate(CASES, start=1):
            par = e & 1
            a0, b0 = _shard(0, p, gen, dt, n)
            a1, b1 = _shard(1, p, gen, dt, n - 5)
            r0, r1 = _additive_partial(p, rep, a0, b0), _additive_partial(p, rep, a1, b1)
            if rank == 1:  # publish rank 1's tagged partial (epoch << 32 | residue) into rank 0's buffer
                peer[K_SLOTS + par * MAXW + 1] = (e << 32) | r1
                torch.cuda.synchronize()
            dist.barrier()
            if rank == 0:
                ta, tb = torch.from_numpy(a0).cuda(), torch.from_numpy(b0).cuda()
                got = gd.dot_fused(ta, tb, p, rep, x).cpu()
                torch.cuda.synchronize()
                total = (r0 + r1) % p
                if rep == 1:
                    want = total  # the sum of Montgomery forms is the Montgomery form of the sum
                elif rep == 3:
                    want = oracle.zech_encode(p, 2, total) if total else 0
                else:
                    want = total
                val = got[0].item() if got.dtype == torch.float64 else int(got.to(torch.int64)[0])
                assert val == want, (e, p, rep, val, want)
                assert int(mine[0].item()) == e, "own epoch word"
            dist.barrier()
            if rank == 1:  # rank 0's kernel stored its tagged partial into THIS process's buffer
                assert int(mine[K_SLOTS + par * MAXW + 0].item()) == (e << 32) | r0, (e, "slot")
                assert int(mine[0].item()) == 0, "a peer never writes the epoch word"
            dist.barrier()
        torch.cuda.synchronize()
        x.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as ex:  # noqa: BLE001 -- report every failure to the parent
        import traceback
        q.put((rank, "".join(traceback.format_exception(ex))))


@pytest.mark.timeout(300)
def test_fused_combine_across_processes_ipc():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in procs:
        r, msg = q.get(timeout=280)
        res[r] = msg
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
