"""Multi-GPU layer: shard long vectors (or batch rows) across ranks, one process per GPU.

Single dot: rank g owns the contiguous slice [g n / G, (g+1) n / G) of both operands,
computes its partial residue with gfp_dot_partial (one kernel), the partials are summed with ONE
all_reduce(SUM) of a single int64 over NCCL (NVLink / NVSwitch), and gfp_finalize reduces mod p and
encodes (one tiny kernel).  Partials are residues < p < 2^32 in the representation's additive form
(classical value, Montgomery form -- the representation is linear --, fp64 integer, Zech classical value),
so the int64 sum of up to 2^31 ranks cannot overflow.

Fused variant: `PeerExchange` maps every rank's small exchange buffer into every process
(CUDA IPC over NVLink; handles exchanged once with all_gather_object), and `dot_fused` runs ONE kernel per
rank whose last CTA stores the shard partial into every peer's buffer, waits for all peers' partials and
finalizes (gfp_dot_allreduce) -- no NCCL launch, no separate finalize.

Batch (matrix-vector): rows are independent, so rank g owns a contiguous row block and there is no
collective on the data path ("weak" in the sense of no exchange); the output stays sharded unless
gather=True asks for an all_gather.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import dot_allreduce as _dot_allreduce
from . import dot_batch as _dot_batch
from . import dot_partial as _dot_partial
from . import finalize as _finalize


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of rank's contiguous shard; shards differ in size by at most one element."""
    if world <= 0 or not 0 <= rank < world or n < 0:
        raise ValueError("need world > 0, 0 <= rank < world, n >= 0")
    return n * rank // world, n * (rank + 1) // world


def combine_partials(partial: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank int64 partial residues in place (one all_reduce of 8 bytes)."""
    if partial.dtype != torch.int64 or partial.numel() != 1:
        raise ValueError("partial must be a 1-element int64 tensor")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return partial


class _LibXchg:
    """The library's exchange-buffer calls (the default backend of PeerExchange)."""

    @staticmethod
    def create():
        from . import xchg_create
        return xchg_create()

    @staticmethod
    def open(handle):
        from . import xchg_open
        return xchg_open(handle)

    @staticmethod
    def close(ptr):
        from . import xchg_close
        xchg_close(ptr)

    @staticmethod
    def destroy(ptr):
        from . import xchg_destroy
        xchg_destroy(ptr)


class PeerExchange:
    """Exchange buffers of a process group for the fused combine: this rank creates one, the IPC handles
    are all-gathered (host objects), every peer's buffer is mapped here, and `spec` is the gfp_xchg the
    kernel needs (peers in rank order, this rank's own pointer at its own index).  `backend` provides
    create() -> (ptr, handle), open(handle) -> ptr, close(ptr), destroy(ptr) (injectable for tests)."""

    def __init__(self, group=None, backend=None):
        from . import XCHG_MAX_WORLD, GfpXchg
        self.backend = backend or _LibXchg
        init = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if init else 1
        self.rank = dist.get_rank(group) if init else 0
        if self.world > XCHG_MAX_WORLD:
            raise ValueError(f"the fused combine supports up to {XCHG_MAX_WORLD} ranks")
        self.own, handle = self.backend.create()
        handles = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(handles, (self.rank, handle), group=group)
        else:
            handles = [(0, handle)]
        if [r for r, _ in handles] != list(range(self.world)):
            raise RuntimeError("exchange handles arrived out of rank order")
        self.ptrs = []
        self.opened = []
        for r, h in handles:
            if r == self.rank:
                self.ptrs.append(self.own)
            else:
                ptr = self.backend.open(h)
                self.ptrs.append(ptr)
                self.opened.append(ptr)
        self.spec = GfpXchg()
        self.spec.rank, self.spec.world = self.rank, self.world
        for r, ptr in enumerate(self.ptrs):
            self.spec.peers[r] = ptr
        self.group = group

    def check(self, device, seconds: float = 10.0) -> bool:
        """Connectivity check before relying on the group: one fused dot of a tiny input with a SOFT timeout armed
        (gfp_xchg_soft_timeout), so a peer whose stores never arrive is reported here as False instead of
        trapping the kernel.  Every rank of the group must call it (it is one collective epoch)."""
        from . import CLASSICAL, dot_allreduce, xchg_soft_timeout, xchg_timed_out
        xchg_soft_timeout(self.own, int(seconds * 1e9))
        try:
            t = torch.ones(1024, dtype=torch.uint32, device=device)
            dot_allreduce(t, t, 65521, CLASSICAL, self.spec)
            torch.cuda.synchronize(device)
            return not xchg_timed_out(self.own)
        finally:
            xchg_soft_timeout(self.own, 0)

    def close(self):
        """Unmap the peers' buffers, wait for every rank to have done the same, free this rank's buffer."""
        for ptr in self.opened:
            self.backend.close(ptr)
        self.opened = []
        if self.world > 1:
            dist.barrier(group=self.group)
        if self.own is not None:
            self.backend.destroy(self.own)
            self.own = None


class _LibMc:
    """The library's multicast calls (the default backend of MulticastExchange)."""

    @staticmethod
    def create(world):
        from . import mc_create
        return mc_create(world)

    @staticmethod
    def import_(fd, nbytes, world):
        from . import mc_import
        return mc_import(fd, nbytes, world)

    @staticmethod
    def add_device(h):
        from . import mc_add_device
        mc_add_device(h)

    @staticmethod
    def bind(h):
        from . import mc_bind
        mc_bind(h)

    @staticmethod
    def destroy(h):
        from . import mc_destroy
        mc_destroy(h)


def _pass_fd(fd, group, rank, world, tag):
    """Rank 0's file descriptor to every other rank of the group (SCM_RIGHTS over a Unix socket whose path is
    broadcast with the process group); returns the descriptor as received here (rank 0: its own)."""
    import os
    import socket
    import tempfile
    path = [None]
    if rank == 0:
        path[0] = os.path.join(tempfile.gettempdir(), f"gfp_mc_{os.getpid()}_{tag}.sock")
        if os.path.exists(path[0]):
            os.unlink(path[0])
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(path[0])
        srv.listen(world)
    dist.broadcast_object_list(path, src=0, group=group)
    if rank == 0:
        try:
            for _ in range(world - 1):
                conn, _ = srv.accept()
                with conn:
                    socket.send_fds(conn, [b"f"], [fd])
                    conn.recv(1)  # the peer holds its copy of the descriptor
        finally:
            srv.close()
            os.unlink(path[0])
        return fd
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    cli.connect(path[0])
    with cli:
        _, fds, _, _ = socket.recv_fds(cli, 1, 1)
        cli.sendall(b"k")
    return fds[0]


class MulticastExchange:
    """The NVLS multicast buffer of a process group for dot_fused_mc (include/gfp.h, gfp_mc_*): rank 0 creates
    the multicast object and passes its descriptor to the others, every rank adds its device, then -- after a
    group barrier -- backs and maps it; `handle` is what the kernel launch needs.  `backend` provides create,
    import_, add_device, bind, destroy (injectable for tests)."""

    def __init__(self, group=None, backend=None):
        self.backend = backend or _LibMc
        init = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if init else 1
        self.rank = dist.get_rank(group) if init else 0
        self.group = group
        info = [None, None]
        if self.rank == 0:
            self.handle, fd, nbytes = self.backend.create(self.world)
            info = [fd, nbytes]
        if self.world > 1:
            dist.broadcast_object_list(info, src=0, group=group)  # (rank 0's fd number is meaningless elsewhere)
            fd = _pass_fd(info[0] if self.rank == 0 else None, group, self.rank, self.world, tag=id(self))
            if self.rank != 0:
                import os
                try:
                    self.handle = self.backend.import_(fd, info[1], self.world)
                finally:
                    os.close(fd)  # the imported handle does not need the descriptor
        self.backend.add_device(self.handle)
        if self.world > 1:
            dist.barrier(group=group)  # every device added before any rank binds memory
        self.backend.bind(self.handle)
        if self.world > 1:
            dist.barrier(group=group)  # every copy zeroed before any rank's first reduction

    def close(self):
        if self.world > 1:
            dist.barrier(group=self.group)
        if self.handle is not None:
            self.backend.destroy(self.handle)
            self.handle = None


def dot_fused(a_shard: torch.Tensor, b_shard: torch.Tensor, p: int, rep: int, xchg,
              out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Exact dot of the globally sharded vectors in ONE kernel launch per rank (compute + exchange +
    finalize); every rank receives the result (device, 1 element).  `xchg` is a PeerExchange (peer stores
    over NVLink) or a MulticastExchange (NVLS multimem reductions in the switch)."""
    if isinstance(xchg, MulticastExchange):
        from . import dot_allreduce_mc
        return dot_allreduce_mc(a_shard, b_shard, p, rep, xchg.handle, out=out, stream=stream)
    return _dot_allreduce(a_shard, b_shard, p, rep, xchg.spec, out=out, stream=stream)


def dot(a_shard: torch.Tensor, b_shard: torch.Tensor, p: int, rep: int, group=None,
        out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Exact dot of the globally sharded vectors; every rank receives the result (device, 1 element).

    With `stream`, the three steps run on it: the all_reduce is issued while `stream` is torch's current
    stream, so NCCL orders itself after the partial kernel and the finalize kernel after the reduction."""
    if stream is None:
        stream = torch.cuda.current_stream(a_shard.device)
    elif not isinstance(stream, torch.cuda.Stream):  # a raw cudaStream_t handle
        stream = torch.cuda.ExternalStream(int(stream), device=a_shard.device)
    with torch.cuda.stream(stream):
        partial = _dot_partial(a_shard, b_shard, p, rep, stream=stream)
        combine_partials(partial, group)
        return _finalize(partial, p, rep, a_shard.dtype, out=out, stream=stream)


def dot_batch(A_rows: torch.Tensor, x: torch.Tensor, p: int, rep: int, group=None, gather: bool = False,
              stream=None) -> torch.Tensor:
    """This rank's row block of A . x; with gather=True the full output on every rank (all_gather)."""
    out = _dot_batch(A_rows, x, p, rep, stream=stream)
    if not gather or not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return out
    world = dist.get_world_size(group)
    sizes = torch.tensor([out.numel()], dtype=torch.int64, device=out.device)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    m = int(max(s.item() for s in all_sizes))
    buf = torch.zeros(m, dtype=torch.int64, device=out.device)
    buf[:out.numel()] = out.to(torch.int64)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([pt[:int(s.item())] for pt, s in zip(parts, all_sizes)]).to(out.dtype)
