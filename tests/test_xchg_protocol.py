"""Host-side checks of the fused multi-GPU combine (gfp_dot_allreduce; SURVEY 8(e) fused variant).

1. A model of the device protocol (xchg_allreduce in kernels_common.cuh, step for step): R ranks as threads with
   random delays between every step run many epochs on shared "exchange buffers"; every rank must obtain
   the exact sum of all ranks' partials at every epoch.  This exercises the two-slot (epoch parity)
   argument of gfp.h: a rank can only overwrite epoch e's slots after every rank has read them.
2. PeerExchange's host logic over gloo (world_size 2, 127.0.0.1) with an injected buffer backend: peers in
   rank order, the own buffer at the own index, every foreign handle opened once, close/destroy order.
"""
import os
import random
import socket
import threading
import time

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

MAXW = 16
XSLOTS = 8 + 2 * MAXW


def model_allreduce(bufs, rank, world, r, p, jitter):
    """The kernel's xchg_allreduce on Python lists (one list of words per rank's buffer): one tagged word
    (epoch << 32 | residue) per slot, written in a single store, polled until the tag matches."""
    own = bufs[rank]
    e = own[0] + 1
    par = e & 1
    tag = e & 0xFFFFFFFF
    assert 0 <= r < 2 ** 32
    for q in range(world):
        jitter()
        bufs[q][XSLOTS + par * MAXW + rank] = (tag << 32) | r  # one single-copy-atomic 64-bit store
    total = 0
    for q in range(world):
        deadline = time.time() + 20
        while True:
            v = own[XSLOTS + par * MAXW + q]
            if v >> 32 == tag:
                break
            if time.time() > deadline:
                raise TimeoutError(f"rank {rank} epoch {e}: peer {q} never arrived")
            time.sleep(0)
        jitter()
        total += v & 0xFFFFFFFF
    own[0] = e
    return total % p


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_protocol_model_many_epochs(world):
    p, epochs = 2 ** 31 - 1, 150
    bufs = [[0] * (8 + 4 * MAXW) for _ in range(world)]
    rng = [random.Random(1000 * world + r) for r in range(world)]
    partial = [[rng[r].randrange(p) for _ in range(epochs)] for r in range(world)]
    results = [[None] * epochs for _ in range(world)]
    errors = []

    def run(rank):
        g = random.Random(rank + 7)

        def jitter():
            if g.random() < 0.3:
                time.sleep(g.random() * 1e-4)
        try:
            for ep in range(epochs):
                results[rank][ep] = model_allreduce(bufs, rank, world, partial[rank][ep], p, jitter)
        except Exception as ex:  # pragma: no cover - surfaced below
            errors.append(repr(ex))

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for ep in range(epochs):
        want = sum(partial[r][ep] for r in range(world)) % p
        assert [results[r][ep] for r in range(world)] == [want] * world, ep
    assert all(b[0] == epochs for b in bufs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class FakeBackend:
    def __init__(self, rank):
        self.rank, self.log = rank, []

    def create(self):
        self.log.append(("create",))
        return 1000 + self.rank, b"h%d" % self.rank

    def open(self, handle):
        self.log.append(("open", handle))
        return 2000 + int(handle[1:])

    def close(self, ptr):
        self.log.append(("close", ptr))

    def destroy(self, ptr):
        self.log.append(("destroy", ptr))


def _worker(rank, world, port, q):
    try:
        from paper_cs_0404008_b200 import dist as gd
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        be = FakeBackend(rank)
        x = gd.PeerExchange(backend=be)
        peers = [x.spec.peers[i] for i in range(world)]
        spec = (x.spec.rank, x.spec.world, peers)
        x.close()
        q.put((rank, spec, be.log, None))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, None, None, repr(e)))


def test_peer_exchange_host_logic_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in ps:
        pr.start()
    out = {}
    for _ in range(world):
        rank, spec, log, err = q.get(timeout=120)
        assert err is None, err
        out[rank] = (spec, log)
    for pr in ps:
        pr.join(timeout=60)
    assert out[0][0] == (0, 2, [1000, 2001])
    assert out[1][0] == (1, 2, [2000, 1001])
    assert out[0][1] == [("create",), ("open", b"h1"), ("close", 2001), ("destroy", 1000)]
    assert out[1][1] == [("create",), ("open", b"h0"), ("close", 2000), ("destroy", 1001)]


def test_peer_exchange_single_process():
    from paper_cs_0404008_b200 import dist as gd
    be = FakeBackend(0)
    x = gd.PeerExchange(backend=be)
    assert (x.spec.rank, x.spec.world, x.spec.peers[0]) == (0, 1, 1000)
    x.close()
    assert be.log == [("create",), ("destroy", 1000)]
