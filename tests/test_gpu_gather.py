"""GPU tests of the fused compute + all-gather entry points (include/ragged_dist.h,
SURVEY.md §8(e)).

The multi-rank exchange is exercised on ONE GPU: "ranks" are launches on
separate CUDA streams and "peer" buffers are local allocations, so the same
kernel code (multi-destination stores, system-scope release/acquire signals,
the last-CTA barrier) runs as on an NVLink box, where the only difference is
that out[r] / signal[r] are peer-mapped pointers.

Parity: gathered rows are bitwise equal to the single-GPU
ragged_pack_attend_unpack / ragged_attn rows on the same inputs (the gather
changes only where rows are stored), which are themselves pinned to the fp64
oracle in test_gpu_parity.py; one case is also checked against the oracle
directly."""
import numpy as np
import pytest
import torch

import synth
from helpers import bits, check_attention, fused_oracle, to_np

rb = pytest.importorskip("paper_2604_15408_b200")
pytestmark = pytest.mark.gpu
DEV = "cuda"
SENT = -12345  # int16 sentinel bit pattern for "never written"


def _inputs(B, N, H, p, seed=0, dtype="bf16", method="l2"):
    q, k, v, keep = synth.make_inputs(B, N, H, p, method, dtype, seed=seed)
    return [t.to(DEV) for t in (q, k, v, keep)]


def _sentinel(shape, dtype):
    t = torch.empty(shape, dtype=dtype, device=DEV)
    t.view(torch.int16).fill_(SENT)
    return t


def _elem_ptr(t, elems):
    return t.data_ptr() + elems * t.element_size()


def test_world1_equals_fused_and_cls_rows():
    B, N, H = 9, 197, 12
    q, k, v, keep = _inputs(B, N, H, 0.7, seed=3)
    keep[4, 0] = 0                                  # a dropped CLS -> +0 CLS row
    keep[6] = 0                                     # an empty image
    ref, rcu = rb.pack_attend_unpack(q, k, v, keep, want_cu=True)
    o = _sentinel((B, N, H, 64), q.dtype)
    cls = _sentinel((B, H * 64), q.dtype)
    cu = torch.empty(B + 1, dtype=torch.int32, device=DEV)
    rb.pack_attend_unpack_gather(q, k, v, keep, rb.gather_desc(1, 0, out=[o], cls=[cls]), cu=cu)
    torch.cuda.synchronize()
    assert (bits(o) == bits(ref)).all()
    assert (bits(cls) == bits(ref[:, 0].reshape(B, H * 64))).all()
    assert (bits(cls[4]) == 0).all() and (bits(cls[6]) == 0).all()
    assert cu.tolist() == rcu.tolist()
    got, _ = fused_oracle(q, k, v, keep)
    check_attention(to_np(o), got, q.dtype)


def test_cls_only_writes_no_padded_rows():
    B, N, H = 5, 197, 3
    q, k, v, keep = _inputs(B, N, H, 0.5, seed=4)
    ref = rb.pack_attend_unpack(q, k, v, keep)
    cls = _sentinel((B, H * 64), q.dtype)
    rb.pack_attend_unpack_gather(q, k, v, keep, rb.gather_desc(1, 0, cls=[cls]))
    torch.cuda.synchronize()
    assert (bits(cls) == bits(ref[:, 0].reshape(B, H * 64))).all()


@pytest.mark.parametrize("world,rank", [(3, 1), (8, 5)])
def test_multi_destination_shards(world, rank):
    """One rank's shard lands at its offset in every destination; the rest of
    every destination is untouched."""
    Bg, N, H = 12, 197, 4
    off, B = rb_shard(Bg, world, rank)
    q, k, v, keep = _inputs(Bg, N, H, 0.6, seed=5)
    ref = rb.pack_attend_unpack(q, k, v, keep)
    qs, ks, vs, kps = (t[off:off + B].contiguous() for t in (q, k, v, keep))
    dests = [_sentinel((Bg, N, H, 64), q.dtype) for _ in range(world)]
    clss = [_sentinel((Bg, H * 64), q.dtype) for _ in range(world)]
    g = rb.gather_desc(world, rank, out=[_elem_ptr(d, off * N * H * 64) for d in dests],
                       cls=[_elem_ptr(c, off * H * 64) for c in clss])
    rb.pack_attend_unpack_gather(qs, ks, vs, kps, g)
    torch.cuda.synchronize()
    for d, c in zip(dests, clss):
        assert (bits(d[off:off + B]) == bits(ref[off:off + B])).all()
        assert (bits(d[:off]) == SENT).all() and (bits(d[off + B:]) == SENT).all()
        assert (bits(c[off:off + B]) == bits(ref[off:off + B, 0].reshape(B, H * 64))).all()
        assert (bits(c[:off]) == SENT).all() and (bits(c[off + B:]) == SENT).all()


def rb_shard(Bg, world, rank):
    from paper_2604_15408_b200.shard import shard
    return shard(Bg, world, rank)


def _host_delay():
    import time
    time.sleep(0.2)


def _virtual_ranks_fused(world, Bg, N, H, p, iters=3, delay_rank=None, want_cu=False, seed=6,
                         delay_fn=_host_delay):
    """`world` ranks as launches on separate streams, each writing its shard
    into every rank's gathered buffer, with the signal barrier."""
    q, k, v, keep = _inputs(Bg, N, H, p, seed=seed)
    ref = rb.pack_attend_unpack(q, k, v, keep)
    gathered = [_sentinel((Bg, N, H, 64), q.dtype) for _ in range(world)]
    sig = [torch.zeros(world, dtype=torch.int32, device=DEV) for _ in range(world)]
    state = [torch.zeros(2, dtype=torch.int32, device=DEV) for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    shards = [rb_shard(Bg, world, r) for r in range(world)]
    parts = [tuple(t[o:o + b].contiguous() for t in (q, k, v, keep)) for o, b in shards]
    cus = [torch.empty(b + 1, dtype=torch.int32, device=DEV) if want_cu else None for _, b in shards]
    torch.cuda.synchronize()
    for it in range(iters):
        for gb in gathered:
            gb.view(torch.int16).fill_(SENT)
        torch.cuda.synchronize()
        for r in range(world):
            off, b = shards[r]
            g = rb.gather_desc(world, r, out=[_elem_ptr(gb, off * N * H * 64) for gb in gathered],
                               signal=sig, state=state[r])
            if r == delay_rank:
                delay_fn()   # the others' last CTAs must wait for this rank
            with torch.cuda.stream(streams[r]):
                rb.pack_attend_unpack_gather(*parts[r], g, cu=cus[r], stream=streams[r])
        torch.cuda.synchronize()
        for gb in gathered:
            assert (bits(gb) == bits(ref)).all(), f"iteration {it}"
        for r in range(world):
            assert state[r].tolist() == [0, it + 1]              # counter reset, epoch advanced
            assert sig[r].tolist() == [it + 1] * world
    if want_cu:
        for (off, b), cu in zip(shards, cus):
            _, rcu = rb.pack_attend_unpack(*(t[off:off + b].contiguous() for t in (q, k, v, keep)),
                                           want_cu=True)
            assert cu.tolist() == rcu.tolist()


def test_virtual_ranks_barrier_two():
    _virtual_ranks_fused(2, 16, 197, 12, 0.8)


def test_virtual_ranks_barrier_late_peer():
    """One rank's launch comes 200 ms late (host delay, as a slow peer process
    would): the others' last CTAs wait in the barrier, and every gathered
    buffer is complete.  (A delay made with a spin kernel on this GPU is not
    equivalent: the GPU's own stream scheduling may then serialise the late
    rank behind the waiting ones -- a single-GPU artifact, not a peer.)"""
    _virtual_ranks_fused(3, 12, 197, 6, 0.5, iters=2, delay_rank=2)


def test_virtual_ranks_barrier_with_scan_cta():
    """B*N > 65536: the extra cu_seqlens scan CTA also counts into the barrier."""
    _virtual_ranks_fused(2, 700, 197, 1, 0.7, iters=2, want_cu=True)


def test_virtual_ranks_packed_gather():
    """ragged_attn_gather: each rank's packed O rows land in its capacity slot
    (first image * N rows) of every rank's gathered packed buffer."""
    world, Bg, N, H = 2, 10, 197, 12
    q, k, v, keep = _inputs(Bg, N, H, 0.7, seed=8)
    gathered = [_sentinel((Bg * N, H, 64), q.dtype) for _ in range(world)]
    sig = [torch.zeros(world, dtype=torch.int32, device=DEV) for _ in range(world)]
    state = [torch.zeros(2, dtype=torch.int32, device=DEV) for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    refs = []
    packed = []
    for r in range(world):
        off, b = rb_shard(Bg, world, r)
        qp, kp, vp, cu, _, _ = rb.pack(*(t[off:off + b].contiguous() for t in (q, k, v, keep)))
        refs.append((off, b, cu, rb.attn(qp, kp, vp, cu, N)))
        packed.append((qp, kp, vp, cu))
    torch.cuda.synchronize()
    for r in range(world):
        off, b, _, _ = refs[r]
        g = rb.gather_desc(world, r, out=[_elem_ptr(gb, off * N * H * 64) for gb in gathered],
                           signal=sig, state=state[r])
        with torch.cuda.stream(streams[r]):
            rb.attn_gather(*packed[r], N, g, stream=streams[r])
    torch.cuda.synchronize()
    for gb in gathered:
        for off, b, cu, op in refs:
            T = int(cu[-1])
            assert (bits(gb[off * N:off * N + T]) == bits(op[:T])).all()
            assert (bits(gb[off * N + T:(off + b) * N]) == SENT).all()


def test_tcgen05_engine_rejected():
    q, k, v, keep = _inputs(2, 197, 3, 0.5)
    o = torch.empty(2, 197, 3, 64, dtype=q.dtype, device=DEV)
    with pytest.raises(rb.RaggedError) as e:
        rb.pack_attend_unpack_gather(q, k, v, keep, rb.gather_desc(1, 0, out=[o]),
                                     engine=rb.ENGINE_TCGEN05)
    assert e.value.status == rb.ENOTSUP


def test_library_nccl_allgather_world1_bitwise():
    """The library's NCCL exchange (ragged_dist.h, NCCL dlopen'ed at run time)
    with a world-1 communicator: the shard's rows land in o_all / cls_all
    bitwise equal to ragged_pack_attend_unpack's, and the call graph-captures."""
    if not rb.nccl_available():
        pytest.skip("NCCL not loadable")
    B, N, H = 6, 197, 12
    q, k, v, keep = _inputs(B, N, H, 0.7, seed=21)
    keep[2, 0] = 0
    ref = rb.pack_attend_unpack(q, k, v, keep)
    comm = rb.NcclComm(rb.nccl_unique_id(), 1, 0)
    o_all = _sentinel((B, N, H, 64), q.dtype)
    cls_all = _sentinel((B, H * 64), q.dtype)
    cu = torch.empty(B + 1, dtype=torch.int32, device=DEV)
    rb.pack_attend_unpack_allgather(q, k, v, keep, comm, o_all, cls_all=cls_all, cu=cu)
    torch.cuda.synchronize()
    assert (bits(o_all) == bits(ref)).all()
    assert (bits(cls_all) == bits(ref[:, 0].reshape(B, H * 64))).all()
    cls2 = _sentinel((B, H * 64), q.dtype)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        rb.cls_allgather(q, k, v, keep, comm, cls2)
    g.replay()
    torch.cuda.synchronize()
    assert (bits(cls2) == bits(cls_all)).all()
    comm.close()


@pytest.mark.parametrize("n_hint", [0, 39, 197])
def test_gather_kernel_variant_follows_n_hint(n_hint):
    """the gather entry points pick the same kernel variant as the
    local call for the same prob (the long-sequence variant for n_hint > 64),
    so the gathered rows are bitwise those of ragged_pack_attend_unpack and of
    ragged_attn on the mma.sync engine with that n_hint."""
    B, N, H = 6, 197, 12
    q, k, v, keep = _inputs(B, N, H, 0.0 if n_hint == 197 else 0.8, seed=31)
    ref = rb.pack_attend_unpack(q, k, v, keep, n_hint=n_hint, engine=rb.ENGINE_MMA_SYNC)
    o = _sentinel((B, N, H, 64), q.dtype)
    rb.pack_attend_unpack_gather(q, k, v, keep, rb.gather_desc(1, 0, out=[o]), n_hint=n_hint)
    qp, kp, vp, cu, _, _ = rb.pack(q, k, v, keep)
    # the gather kernels run the mma.sync engine: compare with ragged_attn on that
    # engine (AUTO takes the warp-specialised engine at n_hint > 148)
    refp = rb.attn(qp, kp, vp, cu, N, n_hint=n_hint, engine=rb.ENGINE_MMA_SYNC)
    op = _sentinel((B * N, H, 64), q.dtype)
    rb.attn_gather(qp, kp, vp, cu, N, rb.gather_desc(1, 0, out=[op]), n_hint=n_hint)
    torch.cuda.synchronize()
    T = int(cu[-1].item())
    assert (bits(o) == bits(ref)).all()
    assert (bits(op[:T]) == bits(refp[:T])).all()
