"""Batch sharding for the multi-GPU path.

Every (image, head) problem is independent (Alg. 1 reads only its own rows,
P:329), so the batch is partitioned into contiguous image ranges, one per rank,
with no data-path collective.  The optional exchange step is an all-gather of
the per-rank outputs (BASELINE.json north_star: "NCCL used only to all-gather
outputs").  Host plumbing only: the compute is the C ABI on each rank's GPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(B_global: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced partition: (first image, number of images) of `rank`.
    The first B_global % world ranks get one extra image."""
    if world < 1 or not (0 <= rank < world) or B_global < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(B_global, world)
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, count


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_gather_images(local: torch.Tensor, B_global: int) -> torch.Tensor:
    """All-gather per-rank [count, ...] outputs into [B_global, ...] on every
    rank (ranks' shards from `shard`, padded to equal size for the collective)."""
    world = dist.get_world_size()
    per = -(-B_global // world)
    pad = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad)
    parts = []
    for r in range(world):
        off, cnt = shard(B_global, world, r)
        parts.append(out[r * per: r * per + cnt])
    return torch.cat(parts, 0)
