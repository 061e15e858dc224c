"""World-size-2 gloo tests of the sharded path's host logic (CPU, no GPU):
shards partition the batch, per-image seeding makes each rank's inputs equal
the global slice, max-over-ranks timing, and the all-gathered outputs equal
the single-process result bit for bit.  The per-rank compute here is the fp64
oracle (tests may call it); on the GPU box the same plumbing wraps the C ABI."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_15408_b200.shard import (all_gather_images, broadcast_bytes, max_over_ranks, packed_capacity, shard,
                                        weak_shard)


def test_shard_partition():
    for B in (0, 1, 7, 32, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                off, cnt = shard(B, world, r)
                seen.extend(range(off, off + cnt))
            assert seen == list(range(B))
            counts = [shard(B, world, r)[1] for r in range(world)]
            assert max(counts) - min(counts) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, q_ref):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    off, cnt = shard(B, world, rank)
    q, k, v, keep = synth.make_inputs(cnt, 41, 2, 0.6, "l2", "bf16", seed=3, image_offset=off)
    # 1) inputs of this rank == the global slice (bitwise)
    assert torch.equal(q.view(torch.int16), q_ref[off:off + cnt].view(torch.int16))
    # 2) per-rank compute, then the exchange step
    o, _ = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    gathered = all_gather_images(torch.from_numpy(o), B)
    # 3) timing = max over ranks
    t = max_over_ranks(1.0 + rank)
    dist.barrier()
    dist.destroy_process_group()
    return gathered, t


def _entry(rank, world, port, B, q_ref, out_q):
    g, t = _worker(rank, world, port, B, q_ref)
    out_q.put((rank, g.numpy(), t))


@pytest.mark.parametrize("B", [6, 7])
def test_two_rank_gather_equals_single_process(B):
    import oracle
    import synth
    q, k, v, keep = synth.make_inputs(B, 41, 2, 0.6, "l2", "bf16", seed=3)
    ref, _ = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_entry, args=(r, 2, port, B, q, out_q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, g, t in res:
        assert np.array_equal(g, ref)        # bitwise: same inputs, same arithmetic
        assert t == 2.0                      # max over ranks


def _ragged(keep, off):
    """Per-image token counts that differ across ranks: image g drops its last
    g % 5 kept tokens (deterministic in the global image index)."""
    keep = keep.clone()
    for i in range(keep.shape[0]):
        idx = torch.nonzero(keep[i]).flatten()
        drop = (off + i) % 5
        if drop:
            keep[i, idx[-drop:]] = 0
    return keep


def _bench_entry(rank, world, port, Bper, out_q):
    """bench.py's N > 1 bookkeeping on gloo: weak-scaling shards of the global
    batch, per-rank inputs equal to the global slice, the packed all-gather
    capacity (max T over ranks), the NCCL unique-id broadcast, max-over-ranks
    timing and the all-gathered outputs of the per-rank compute."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    off, cnt = weak_shard(Bper, world, rank)
    q, k, v, keep = synth.make_inputs(cnt, 33, 2, 0.5, "l2", "bf16", seed=5, image_offset=off)
    keep = _ragged(keep, off)
    T = int(keep.numpy().astype(bool).sum())
    tcap = packed_capacity(T)
    uid = broadcast_bytes(bytes(range(128)) if rank == 0 else None)
    o, _ = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    g = all_gather_images(torch.from_numpy(o), world * Bper)
    t = max_over_ranks(0.5 * (rank + 1))
    dist.barrier()
    dist.destroy_process_group()
    out_q.put((rank, off, cnt, T, tcap, uid, g.numpy(), t))


@pytest.mark.parametrize("world", [2, 4])
def test_bench_sharding_bookkeeping(world):
    import oracle
    import synth
    Bper = 3
    q, k, v, keep = synth.make_inputs(world * Bper, 33, 2, 0.5, "l2", "bf16", seed=5)
    keep = _ragged(keep, 0)
    ref, _ = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_entry, args=(r, world, port, Bper, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(out_q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Ts = [r[3] for r in res]
    kn = keep.numpy().astype(bool)
    for rank, off, cnt, T, tcap, uid, g, t in res:
        assert (off, cnt) == (rank * Bper, Bper)                      # weak scaling: equal shards
        assert T == int(kn[off:off + cnt].sum())                      # data-dependent per-rank T
        assert tcap == max(Ts)
        assert uid == bytes(range(128))
        assert np.array_equal(g, ref)
        assert t == 0.5 * world
