"""Multi-GPU layer: shard long vectors (or batch rows) across ranks, one process per GPU.

Single dot: rank g owns the contiguous slice [g n / G, (g+1) n / G) of both operands,
computes its partial residue with gfp_dot_partial (one kernel), the partials are summed with ONE
all_reduce(SUM) of a single int64 over NCCL (NVLink / NVSwitch), and gfp_finalize reduces mod p and
encodes (one tiny kernel).  Partials are residues < p < 2^32 in the representation's additive form
(classical value, Montgomery form -- the representation is linear --, fp64 integer, Zech classical value),
so the int64 sum of up to 2^31 ranks cannot overflow.

Batch (matrix-vector): rows are independent, so rank g owns a contiguous row block and there is no
collective on the data path ("weak" in the sense of no exchange); the output stays sharded unless
gather=True asks for an all_gather.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

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


def dot(a_shard: torch.Tensor, b_shard: torch.Tensor, p: int, rep: int, group=None,
        out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Exact dot of the globally sharded vectors; every rank receives the result (device, 1 element)."""
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
