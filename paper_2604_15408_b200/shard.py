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


def weak_shard(B_per_rank: int, world: int, rank: int) -> tuple[int, int]:
    """Weak scaling (bench.py): the global batch is world * B_per_rank images;
    this rank's (first image, count) -- every rank holds B_per_rank images, so
    the equal-count all-gathers of ragged_dist.h apply."""
    return shard(world * B_per_rank, world, rank)


def packed_capacity(T_local: int, device=None) -> int:
    """Rows per rank slot of a packed all-gather: the largest rank's live row
    count (ranks' T differ under data-dependent masks)."""
    return int(max_over_ranks(float(T_local), device))


def broadcast_bytes(data: bytes | None, nbytes: int = 128, src: int = 0, device=None) -> bytes:
    """Broadcast an opaque byte string (e.g. the library's NCCL unique id,
    ragged_dist_nccl_unique_id) from rank `src` to every rank."""
    t = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if dist.get_rank() == src:
        if data is None or len(data) != nbytes:
            raise ValueError("source rank must provide nbytes of data")
        t.copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())
