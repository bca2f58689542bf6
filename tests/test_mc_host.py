"""Host logic of the NVLS multicast exchange (paper_cs_0404008_b200.dist.MulticastExchange) on CPU: world_size 2
over gloo with a recording backend in place of the library's gfp_mc_* calls.  Checked: rank 0 alone creates the
multicast object, its file descriptor really crosses to rank 1 (SCM_RIGHTS: rank 1 reads the bytes rank 0 wrote
into the pipe behind it), rank 1 imports it with rank 0's size, every rank adds its device before any rank binds
memory (a barrier between), and destroy runs on every rank.  The device path is tests/test_gpu_parity.py."""
import os
import socket
import time

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

gfp_dist = pytest.importorskip("paper_cs_0404008_b200.dist")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _Rec:
    def __init__(self, rank, log):
        self.rank, self.log = rank, log
        self.r, self.w = os.pipe()

    def create(self, world):
        os.write(self.w, b"mc-object")
        self.log.append(("create", world, time.monotonic()))
        return 1234, self.r, 2 << 20

    def import_(self, fd, nbytes, world):
        data = os.read(fd, 9)
        self.log.append(("import", data.decode(), nbytes, world, time.monotonic()))
        return 5678

    def add_device(self, h):
        self.log.append(("add", h, time.monotonic()))
        time.sleep(0.3 if self.rank == 1 else 0.0)  # a slow rank: the other must wait before binding

    def bind(self, h):
        self.log.append(("bind", h, time.monotonic()))

    def destroy(self, h):
        self.log.append(("destroy", h, time.monotonic()))


def _worker(rank, world, port, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        log = []
        x = gfp_dist.MulticastExchange(backend=_Rec(rank, log))
        handle = x.handle
        x.close()
        dist.destroy_process_group()
        q.put((rank, log, handle, None))
    except Exception as e:  # surface failures in the parent
        q.put((rank, None, None, repr(e)))


def test_multicast_exchange_world2_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(2):
        rank, log, handle, err = q.get(timeout=240)
        assert err is None, err
        out[rank] = (log, handle)
    for pr in procs:
        pr.join(timeout=60)
    log0, h0 = out[0]
    log1, h1 = out[1]
    assert [e[0] for e in log0] == ["create", "add", "bind", "destroy"] and h0 == 1234
    assert [e[0] for e in log1] == ["import", "add", "bind", "destroy"] and h1 == 5678
    assert log0[0][1] == 2
    assert log1[0][1] == "mc-object" and log1[0][2] == 2 << 20 and log1[0][3] == 2  # the fd really crossed
    # nobody binds before every rank added its device (rank 1's add takes 0.3 s)
    last_add = max(log0[1][-1], log1[1][-1])
    assert log0[2][-1] >= last_add and log1[2][-1] >= last_add


def test_multicast_exchange_single_rank():
    log = []
    x = gfp_dist.MulticastExchange(backend=_Rec(0, log))
    assert x.world == 1 and x.handle == 1234
    x.close()
    assert [e[0] for e in log] == ["create", "add", "bind", "destroy"]
