"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Integers (cu_seqlens, dst, src) and copies (pack, unpack) must be bit-exact;
attention within max-abs 2e-3 (bf16) / 5e-4 (fp16) of fp64 (BASELINE.json
north_star; R2).  Sizes span several tiles and ragged tails (n up to
256, partial 16/64-row tiles, empty images); the BASELINE configs C1, C3, C4
are compared in full, C5 (B = 4096) on sampled (image, head) problems plus
properties that hold at any size."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import TOL, bits, check_attention, fused_oracle, to_np

rb = pytest.importorskip("paper_2604_15408_b200")
pytestmark = pytest.mark.gpu
DEV = "cuda"
DT = {"bf16": torch.bfloat16, "fp16": torch.float16}
ENGINES = [rb.ENGINE_MMA_SYNC, rb.ENGINE_TCGEN05]


def _dev(*ts):
    return [t.to(DEV) for t in ts]


# ------------------------------------------------------------------ scan ----

def _scan_case(keep_np):
    keep = torch.from_numpy(keep_np).to(DEV)
    cu, dst, src = rb.scan(keep)
    torch.cuda.synchronize()
    rcu, rdst, rsrc = oracle.scan(keep_np)
    T = int(rcu[-1])
    assert cu.cpu().numpy().tolist() == rcu.tolist()
    assert dst.cpu().numpy().tolist() == rdst.tolist()
    assert src[:T].cpu().numpy().tolist() == rsrc[:T].tolist()


def test_scan_spec_example():
    _scan_case(np.array([[1, 0, 1], [1, 1, 1]], np.uint8))


@pytest.mark.parametrize("B,N", [(1, 1), (3, 7), (5, 31), (4, 32), (7, 33), (32, 197), (33, 256),
                                 (130, 197), (257, 64), (1000, 197)])
def test_scan_random_masks(B, N):
    rng = np.random.default_rng(B * 1000 + N)
    keep = (rng.random((B, N)) < rng.uniform(0.05, 0.95)).astype(np.uint8)
    keep[rng.random(B) < 0.1] = 0                      # empty images (R11)
    keep[keep == 1] = rng.integers(1, 255, size=int(keep.sum()), dtype=np.uint8)  # nonzero = keep
    _scan_case(keep)


def test_scan_c5_scale_exact():
    keep = synth.mask_threshold_l2(4096, 197, synth.kept_tokens(197, 0.7), seed=1000)
    _scan_case(keep)


@pytest.mark.parametrize("offset", [0, 1, 3])
def test_scan_large_batch_chunked_unaligned(offset):
    """B*N > 65536 takes the chunked scan (one CTA per 16 KB of mask, each
    counting the kept bytes before its chunk): bit-exact for a mask that does
    not start on a 16-byte boundary (byte-load carry path) and for one that
    does, with image boundaries falling inside chunks."""
    B, N = 420, 197
    rng = np.random.default_rng(offset + 7)
    keep_np = (rng.random((B, N)) < 0.45).astype(np.uint8)
    keep_np[rng.random(B) < 0.05] = 0
    buf = torch.zeros(B * N + 16, dtype=torch.uint8)
    buf[offset:offset + B * N] = torch.from_numpy(keep_np.reshape(-1))
    keep = buf.to(DEV)[offset:offset + B * N].view(B, N)
    cu, dst, src = rb.scan(keep)
    torch.cuda.synchronize()
    rcu, rdst, rsrc = oracle.scan(keep_np)
    T = int(rcu[-1])
    assert cu.cpu().numpy().tolist() == rcu.tolist()
    assert dst.cpu().numpy().tolist() == rdst.tolist()
    assert src[:T].cpu().numpy().tolist() == rsrc[:T].tolist()


# ------------------------------------------------------------------ pack ----

@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("B,N,H,p", [(4, 197, 3, 0.5), (3, 33, 2, 0.3), (32, 197, 12, 0.8), (2, 256, 4, 0.0)])
def test_pack_bitwise(dtype, B, N, H, p):
    q, k, v, keep = synth.make_inputs(B, N, H, p, "l2", dtype, seed=1)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    qp, kp, vp, cu, dst, src = rb.pack(qd, kd, vd, keepd)
    torch.cuda.synchronize()
    rcu, rdst, rsrc = oracle.scan(keep.numpy())
    T = int(rcu[-1])
    assert cu.cpu().tolist() == rcu.tolist()
    for got, x in ((qp, q), (kp, k), (vp, v)):
        assert np.array_equal(bits(got[:T]), oracle.pack(bits(x), rsrc, T))


def test_pack_fused_qkv_layout():
    """ld = 3*H*d: q/k/v are views of one [B, N, 3, H, d] buffer."""
    B, N, H = 5, 197, 6
    qkv = torch.randn(B, N, 3, H, 64, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16)
    keep = torch.from_numpy(synth.mask_random(B, N, 50, seed=4))
    d = qkv.to(DEV)
    q, k, v = d[:, :, 0], d[:, :, 1], d[:, :, 2]
    assert q.stride(1) == 3 * H * 64
    qp, kp, vp, cu, dst, src = rb.pack(q, k, v, keep.to(DEV))
    o = rb.pack_attend_unpack(q, k, v, keep.to(DEV), engine=rb.ENGINE_TCGEN05)
    torch.cuda.synchronize()
    rcu, _, rsrc = oracle.scan(keep.numpy())
    T = int(rcu[-1])
    assert np.array_equal(bits(kp[:T]), oracle.pack(bits(qkv[:, :, 1]), rsrc, T))
    ref, _ = fused_oracle(qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2], keep)
    check_attention(to_np(o), ref, torch.bfloat16, vmax=float(qkv[:, :, 2].float().abs().max()), dist="heavy")


# ------------------------------------------------------------- attention ----

def _attn_case(B, N, H, p, method, dtype, seed, dist="standard", engine=rb.ENGINE_AUTO):
    q, k, v, keep = synth.make_inputs(B, N, H, p, method, dtype, seed=seed, dist=dist)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    qp, kp, vp, cu, dst, src = rb.pack(qd, kd, vd, keepd)
    op = rb.attn(qp, kp, vp, cu, N, engine=engine)
    torch.cuda.synchronize()
    rcu, rdst, rsrc = oracle.scan(keep.numpy())
    T = int(rcu[-1])
    f64 = [oracle.as_f64(t) for t in (q, k, v)]
    ref = oracle.attention(*(oracle.pack(t, rsrc, T) for t in f64), rcu)
    return check_attention(to_np(op[:T]), ref, DT[dtype], vmax=float(v.float().abs().max()), dist=dist)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("B,N,H,p,method", [
    (4, 197, 3, 0.5, "l2"),          # C1
    (6, 197, 2, 0.0, "all"),         # n = 197: 4 kv chunks, 13 query slices, tail 5
    (5, 256, 2, 0.0, "all"),         # maximum N
    (8, 130, 2, 0.5, "random"),      # n = 65: tail of one row
    (8, 129, 3, 0.1, "ats"),         # heterogeneous lengths
    (9, 40, 4, 0.6, "dynamicvit"),
    (3, 17, 2, 0.0, "all"),          # n = 17
])
def test_attn_matches_oracle(engine, dtype, B, N, H, p, method):
    _attn_case(B, N, H, p, method, dtype, seed=2, engine=engine)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("dist", ["peaked", "heavy"])
def test_attn_distributions(engine, dtype, dist):
    _attn_case(6, 197, 3, 0.3, "l2", dtype, seed=5, dist=dist, engine=engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_attn_single_token_and_empty_images(engine):
    """n = 1 -> output is the V row exactly; n = 0 -> no rows written."""
    B, N, H = 6, 31, 2
    q, k, v = synth.activations(B, N, H, 64, "bf16", seed=6)
    keep = np.zeros((B, N), np.uint8)
    keep[0, 0] = 1           # n = 1
    keep[2, [0, 5]] = 1      # n = 2
    keep[4, :] = 1           # n = 31; images 1, 3, 5 empty
    qd, kd, vd = _dev(q, k, v)
    keepd = torch.from_numpy(keep).to(DEV)
    sentinel = torch.full((B, N, H, 64), 7.0, dtype=torch.bfloat16, device=DEV)
    o = rb.pack_attend_unpack(qd, kd, vd, keepd, o=sentinel, engine=engine)
    torch.cuda.synchronize()
    assert torch.equal(o[0, 0].cpu(), v[0, 0])
    for b in (1, 3, 5):
        assert torch.all(o[b] == 0)
    ref, _ = fused_oracle(q, k, v, torch.from_numpy(keep))
    check_attention(to_np(o), ref, torch.bfloat16)


# --------------------------------------------------------------- unpack ----

@pytest.mark.parametrize("B,N,H,p", [(4, 197, 3, 0.5), (7, 100, 5, 0.9), (2, 256, 1, 0.0)])
def test_unpack_bitwise(B, N, H, p):
    q, k, v, keep = synth.make_inputs(B, N, H, p, "random", "fp16", seed=7)
    keep_np = keep.numpy().copy()
    keep_np[B // 2] = 0
    keepd = torch.from_numpy(keep_np).to(DEV)
    cu, dst, src = rb.scan(keepd)
    op = torch.randn(B * N, H, 64, device=DEV).to(torch.float16)
    o = torch.full((B, N, H, 64), 3.0, dtype=torch.float16, device=DEV)
    rb.unpack(op, dst, B, N, o=o)
    torch.cuda.synchronize()
    _, rdst, _ = oracle.scan(keep_np)
    assert np.array_equal(bits(o), oracle.unpack(bits(op), rdst, B, N, 0))


# ----------------------------------------------------------------- fused ----

@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("cfg", ["C1", "C3"])
def test_fused_baseline_configs_full(engine, dtype, cfg):
    c = synth.CONFIGS[cfg]
    H = synth.PRESETS[c["preset"]]["H"]
    q, k, v, keep = synth.make_inputs(c["B"], 197, H, c["p"], c["method"], dtype, seed=0)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    o, cu = rb.pack_attend_unpack(qd, kd, vd, keepd, want_cu=True, engine=engine)
    torch.cuda.synchronize()
    ref, rcu = fused_oracle(q, k, v, keep)
    assert cu.cpu().tolist() == rcu.tolist()
    check_attention(to_np(o), ref, DT[dtype])
    assert np.all(bits(o)[~keep.numpy().astype(bool)] == 0)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("method", ["l2", "dynamicvit", "evit", "ats"])
@pytest.mark.parametrize("p", [0.5, 0.7, 0.9])
def test_fused_c4_generators_full(engine, method, p):
    q, k, v, keep = synth.make_inputs(64, 197, 12, p, method, "bf16", seed=0)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    o = rb.pack_attend_unpack(qd, kd, vd, keepd, engine=engine)
    torch.cuda.synchronize()
    ref, _ = fused_oracle(q, k, v, keep)
    check_attention(to_np(o), ref, torch.bfloat16)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("p", [0.0, 0.3, 0.8])
def test_fused_equals_composed_bitwise(engine, dtype, p):
    """a5 == a4 . a3 . a2 . a1 bit for bit (same arithmetic, same order)."""
    q, k, v, keep = synth.make_inputs(16, 197, 6, p, "ats" if p else "all", dtype, seed=8)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    o1, cu1 = rb.pack_attend_unpack(qd, kd, vd, keepd, want_cu=True, engine=engine)
    qp, kp, vp, cu, dst, src = rb.pack(qd, kd, vd, keepd)
    op = rb.attn(qp, kp, vp, cu, 197, engine=engine)
    o2 = rb.unpack(op, dst, 16, 197)
    torch.cuda.synchronize()
    assert torch.equal(cu1, cu)
    assert np.array_equal(bits(o1), bits(o2))


@pytest.mark.parametrize("engine", ENGINES + [rb.ENGINE_TCGEN05_WS])
def test_graph_replay_and_determinism_bitwise(engine):
    q, k, v, keep = synth.make_inputs(32, 197, 12, 0.8, "l2", "bf16", seed=9)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    o_eager = rb.pack_attend_unpack(qd, kd, vd, keepd, engine=engine)
    o_g = torch.empty_like(o_eager)
    cu_g = torch.empty(33, dtype=torch.int32, device=DEV)
    g = rb.Graph(qd, kd, vd, keepd, o_g, cu_g, engine=engine)
    for _ in range(3):
        o_g.fill_(5.0)
        g.launch()
        torch.cuda.synchronize()
        assert torch.equal(o_g.view(torch.int16), o_eager.view(torch.int16))
    g.close()
    again = rb.pack_attend_unpack(qd, kd, vd, keepd, engine=engine)
    torch.cuda.synchronize()
    assert torch.equal(again.view(torch.int16), o_eager.view(torch.int16))
    assert cu_g.cpu().tolist() == oracle.scan(keep.numpy())[0].tolist()


@pytest.mark.parametrize("engine", ENGINES)
def test_cross_image_isolation_bitwise(engine):
    q, k, v, keep = synth.make_inputs(8, 197, 4, 0.5, "l2", "bf16", seed=10)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    o1 = rb.pack_attend_unpack(qd, kd, vd, keepd, engine=engine)
    kd2, vd2 = kd.clone(), vd.clone()
    kd2[3] = -kd2[3]
    vd2[3] = 0.5 * vd2[3]
    o2 = rb.pack_attend_unpack(qd, kd2, vd2, keepd, engine=engine)
    torch.cuda.synchronize()
    other = [b for b in range(8) if b != 3]
    assert torch.equal(o1[other].view(torch.int16), o2[other].view(torch.int16))
    assert not torch.equal(o1[3], o2[3])


@pytest.mark.parametrize("engine", ENGINES)
def test_constant_v_column_is_exact(engine):
    """A V column equal to c everywhere gives exactly c (checks o / l)."""
    q, k, v, keep = synth.make_inputs(4, 197, 2, 0.0, "all", "bf16", seed=11)
    v[..., 5] = 0.375
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    o = rb.pack_attend_unpack(qd, kd, vd, keepd, engine=engine)
    torch.cuda.synchronize()
    assert torch.all(o[..., 5] == 0.375)


@pytest.mark.parametrize("engine", ENGINES)
def test_c5_scale_sampled(engine):
    """C5 (DeiT-B, B = 4096, 70 %): cu exact in full; zero rows everywhere;
    64 sampled (image, head) problems against the oracle one by one."""
    B, N, H = 4096, 197, 12
    g = torch.Generator(device=DEV).manual_seed(12)
    q = torch.randn(B, N, H, 64, generator=g, device=DEV).to(torch.bfloat16)
    k = torch.randn(B, N, H, 64, generator=g, device=DEV).to(torch.bfloat16)
    v = (torch.rand(B, N, H, 64, generator=g, device=DEV) * 2 - 1).to(torch.bfloat16)
    keep_np = synth.mask_threshold_l2(B, N, synth.kept_tokens(N, 0.7), seed=1012)
    keepd = torch.from_numpy(keep_np).to(DEV)
    o, cu = rb.pack_attend_unpack(q, k, v, keepd, want_cu=True, engine=engine)
    torch.cuda.synchronize()
    assert cu.cpu().numpy().tolist() == oracle.scan(keep_np)[0].tolist()
    dropped = ~keepd.bool()
    assert torch.all(o[dropped] == 0)
    rng = np.random.default_rng(0)
    for b, h in zip(rng.integers(0, B, 64), rng.integers(0, H, 64)):
        pos, rows = oracle.attention_image_head(q[b].cpu()[None], k[b].cpu()[None], v[b].cpu()[None],
                                                keep_np[b][None], 0, int(h))
        got = o[b, torch.from_numpy(pos).to(DEV), int(h)].double().cpu().numpy()
        assert np.abs(got - rows).max() <= TOL[torch.bfloat16]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("B,N", [(9, 197), (5, 33), (400, 197)])  # B*N <= / > 65536: both cu modes
def test_fused_cu_with_empty_images(engine, B, N):
    """cu_seqlens from the fused launch (head-0 prefix mode and scan-CTA mode),
    including empty first / last images, equals the oracle's."""
    rng = np.random.default_rng(B + N)
    keep = (rng.random((B, N)) < 0.3).astype(np.uint8)
    keep[0] = 0
    keep[-1] = 0
    keep[B // 2] = 0
    q, k, v = synth.activations(B, N, 2, 64, "bf16", seed=3)
    qd, kd, vd = _dev(q, k, v)
    o, cu = rb.pack_attend_unpack(qd, kd, vd, torch.from_numpy(keep).to(DEV), want_cu=True, engine=engine)
    torch.cuda.synchronize()
    assert cu.cpu().numpy().tolist() == oracle.scan(keep)[0].tolist()
    assert torch.all(o[0] == 0) and torch.all(o[-1] == 0)


# ------------------------------------------------- N2: on-device prune ----

def _check_l2_mask(x, k, got):
    """Exact where the decision is unique (score gap at the threshold well above
    fp32 rounding); otherwise the result must still be a valid top-k."""
    want = oracle.keep_topk_l2(x, k)
    s = oracle.l2_scores(x)
    B, N = want.shape
    for b in range(B):
        if np.array_equal(got[b], want[b]):
            continue
        srt = np.sort(s[b])[::-1]
        gap = (srt[k - 1] - srt[k]) / srt[k] if 0 < k < N else np.inf
        assert gap < 1e-5, f"image {b}: masks differ although the threshold gap is {gap:.2e}"
        assert got[b].sum() == want[b].sum() and got[b][0] == 1
        assert s[b][got[b] == 1].min() >= s[b][got[b] == 0].max() * (1 - 1e-5)


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("B,N,D,p", [(32, 197, 768, 0.8), (4, 197, 192, 0.5), (7, 33, 64, 0.3),
                                     (3, 256, 384, 0.9), (2, 1, 64, 0.0)])
def test_keep_topk_l2_matches_oracle(dtype, B, N, D, p):
    x = synth.hidden_states(B, N, D, dtype, seed=5)
    k = synth.kept_tokens(N, p)
    keep = rb.keep_topk_l2(x.to(DEV), k)
    torch.cuda.synchronize()
    _check_l2_mask(x, k, keep.cpu().numpy())


def test_keep_topk_l2_ties_and_k_edges():
    """Exact ties resolve to the lower position; k < 1 is rejected (CLS always
    survives), k >= N keeps all; a NaN score ranks last (at most k kept)."""
    x = torch.zeros(2, 9, 64, dtype=torch.bfloat16)
    x[:, 1:, 0] = 1.0                       # all non-CLS scores equal
    x[1, 5, 0] = 2.0
    xd = x.to(DEV)
    got = rb.keep_topk_l2(xd, 4).cpu().numpy()
    assert got[0].tolist() == [1, 1, 1, 1, 0, 0, 0, 0, 0]
    assert got[1].tolist() == [1, 1, 1, 0, 0, 1, 0, 0, 0]
    with pytest.raises(rb.RaggedError):
        rb.keep_topk_l2(xd, 0)
    assert rb.keep_topk_l2(xd, 1).cpu().numpy().tolist() == [[1] + [0] * 8] * 2
    assert rb.keep_topk_l2(xd, 50).cpu().numpy().sum() == 18
    xn = x.clone()
    xn[0, 2, 3] = float("nan")
    got = rb.keep_topk_l2(xn.to(DEV), 4).cpu().numpy()
    assert got[0].tolist() == [1, 1, 0, 1, 1, 0, 0, 0, 0]
    assert got.sum(1).tolist() == [4, 4]


def test_prune_then_fused_path():
    """N2 -> a5: the on-device mask drives the fused path; equals the oracle end to end."""
    B, N, H = 8, 197, 12
    x = synth.hidden_states(B, N, H * 64, "bf16", seed=6)
    q, k, v = synth.activations(B, N, H, 64, "bf16", seed=6)
    keep = rb.keep_topk_l2(x.to(DEV), synth.kept_tokens(N, 0.7))
    o = rb.pack_attend_unpack(*_dev(q, k, v), keep)
    torch.cuda.synchronize()
    km = keep.cpu().numpy()
    _check_l2_mask(x, synth.kept_tokens(N, 0.7), km)
    ref, _ = oracle.pack_attend_unpack(q, k, v, km)
    check_attention(to_np(o), ref, torch.bfloat16)


# ------------------------------------------- a5 from host memory (e2e) ----

@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("B,H,p,method", [(32, 12, 0.8, "l2"), (5, 3, 0.0, "all"), (9, 6, 0.5, "ats")])
def test_fused_host_inputs_bitwise(engine, dtype, B, H, p, method):
    """ragged_pack_attend_unpack_host (pinned host q/k/v/keep read in place by
    the kernel) == the device-resident call, bit for bit, for a device and a
    pinned-host o; cu_seqlens exact; within tolerance of the fp64 oracle."""
    q, k, v, keep = synth.make_inputs(B, 197, H, p, method, dtype, seed=21)
    qh, kh, vh, keeph = (t.pin_memory() for t in (q, k, v, keep))
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    ref, cu_ref = rb.pack_attend_unpack(qd, kd, vd, keepd, want_cu=True, engine=engine)
    o_dev = torch.full_like(ref, 7.0)
    cu_dev = torch.full((B + 1,), -1, dtype=torch.int32, device=DEV)
    rb.pack_attend_unpack_host(qh, kh, vh, keeph, o_dev, cu=cu_dev, engine=engine)
    o_host = torch.full(ref.shape, 7.0, dtype=ref.dtype).pin_memory()
    rb.pack_attend_unpack_host(qh, kh, vh, keeph, o_host, engine=engine)
    torch.cuda.synchronize()
    assert torch.equal(cu_dev, cu_ref)
    assert np.array_equal(bits(o_dev), bits(ref))
    assert np.array_equal(bits(o_host), bits(ref))
    ref64, rcu = fused_oracle(q, k, v, keep)
    assert cu_dev.cpu().numpy().tolist() == np.asarray(rcu).tolist()
    check_attention(to_np(o_dev), ref64, DT[dtype])


def test_fused_host_rejects_pageable():
    q, k, v, keep = synth.make_inputs(2, 197, 3, 0.5, "l2", "bf16", seed=1)
    o = torch.empty(2, 197, 3, 64, dtype=torch.bfloat16, device=DEV)
    p = rb.problem(2, 197, 3)
    st = rb.lib().ragged_pack_attend_unpack_host(
        __import__("ctypes").byref(p), keep.data_ptr(), q.data_ptr(), k.data_ptr(), v.data_ptr(),
        o.data_ptr(), None, None)
    assert st == rb.EINVAL and "pageable" in rb.last_error()


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("B,H,p,method", [(64, 12, 0.5, "ats"), (200, 12, 0.7, "l2"), (150, 3, 0.0, "all"),
                                          (1000, 6, 0.9, "evit")])
def test_fused_large_batch_bitwise(engine, dtype, B, H, p, method):
    """Multi-wave fused launches (more (image, head) problems than resident
    CTAs) equal the composed path (pack -> attn -> unpack) bit for bit; with
    B*N > 65536 cu_seqlens comes from ceil(B/128) concurrent scan items (each
    offsets its group by a streaming count of the preceding images' keeps) and
    must be exact."""
    q, k, v, keep = synth.make_inputs(B, 197, H, p, method, dtype, seed=31)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    o1, cu1 = rb.pack_attend_unpack(qd, kd, vd, keepd, want_cu=True, engine=engine)
    qp, kp, vp, cu, dst, src = rb.pack(qd, kd, vd, keepd)
    o2 = rb.unpack(rb.attn(qp, kp, vp, cu, 197, engine=engine), dst, B, 197)
    torch.cuda.synchronize()
    assert torch.equal(cu1, cu)
    assert cu1.cpu().tolist() == oracle.scan(keep.numpy())[0].tolist()
    assert np.array_equal(bits(o1), bits(o2))
    assert np.all(bits(o1)[~keep.numpy().astype(bool)] == 0)


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("B,N,H,p,method", [(32, 197, 12, 0.0, "all"), (16, 197, 6, 0.3, "l2"), (9, 197, 4, 0.5, "ats"),
                                            (8, 197, 12, 0.8, "l2"), (5, 256, 2, 0.1, "dynamicvit"),
                                            (7, 100, 3, 0.6, "evit"), (400, 197, 2, 0.3, "l2")])
def test_long_sequence_variant(dtype, B, N, H, p, method):
    """ragged_problem.n_hint > 64 selects the mma.sync kernel built for long
    sequences (exact per-chunk tile counts; its straight-line code lets the
    compiler contract different multiply-adds, so bits may differ from the
    default kernel): within tolerance of the fp64 oracle for every n
    (including n <= 64 and an empty image), fused == composed bit for bit under
    the same hint, cu_seqlens exact, and run-to-run deterministic."""
    q, k, v, keep = synth.make_inputs(B, N, H, p, method, dtype, seed=41)
    keep_np = keep.numpy().copy()
    keep_np[B // 2, :] = 0                      # an empty image
    keep = torch.from_numpy(keep_np)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    MMA = rb.ENGINE_MMA_SYNC  # the long variant of the one-stage kernel (AUTO at n_hint >= 188: the WS engine)
    o_long, cu_long = rb.pack_attend_unpack(qd, kd, vd, keepd, want_cu=True, n_hint=N, engine=MMA)
    again = rb.pack_attend_unpack(qd, kd, vd, keepd, n_hint=N, engine=MMA)
    qp, kp, vp, cu, dst, src = rb.pack(qd, kd, vd, keepd)
    # composed path on the fused kernel's engine (AUTO takes the warp-specialised
    # engine at n_hint > 148: equal within tolerance, not bitwise -- tested below)
    o_comp = rb.unpack(rb.attn(qp, kp, vp, cu, N, n_hint=N, engine=rb.ENGINE_MMA_SYNC), dst, B, N)
    o_auto = rb.unpack(rb.attn(qp, kp, vp, cu, N, n_hint=N), dst, B, N)
    torch.cuda.synchronize()
    ref, rcu = fused_oracle(q, k, v, keep)
    assert cu_long.cpu().tolist() == rcu.tolist()
    assert np.array_equal(bits(o_long), bits(o_comp))
    assert np.array_equal(bits(o_long), bits(again))
    check_attention(to_np(o_long), ref, DT[dtype])
    check_attention(to_np(o_auto), ref, DT[dtype])
    assert np.all(bits(o_long)[~keep_np.astype(bool)] == 0)


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("ramp", [0.0, 5.0, 40.0, -40.0])
def test_long_variant_running_max_paths(dtype, ramp):
    """Scores that rise across the 64-key chunks exercise both branches of the
    long kernel's lazy rescaling (Alg. 1 lines 10-13): ramp 5 keeps
    every later chunk max within 2^8 of the first (no rescale after chunk 0,
    P up to ~2^5), ramp 40 raises the max by ~13 nats per chunk (rescale every
    chunk), -40 puts the max in chunk 0.  q = 8e, k_n = ramp*(n/N)*e + noise with
    e.e = 1, so the score of key n is ~ramp*n/N nats.  Both kernels within
    tolerance of the fp64 oracle; fused == composed bitwise under the hint."""
    B, N, H = 6, 197, 3
    q, k, v, keep = synth.make_inputs(B, N, H, 0.0, "all", dtype, seed=77)
    e = torch.full((64,), 1.0 / 8.0)
    g = torch.Generator().manual_seed(5)
    pos = (torch.arange(N, dtype=torch.float32) / N).view(1, N, 1, 1)
    tdt = q.dtype
    qf = 8.0 * e.view(1, 1, 1, 64) + 0.3 * torch.randn(B, N, H, 64, generator=g)
    kf = ramp * pos * e.view(1, 1, 1, 64) + 0.3 * torch.randn(B, N, H, 64, generator=g)
    q, k = qf.to(tdt), kf.to(tdt)
    keep_np = keep.numpy().copy()
    keep_np[1, 150:] = 0                       # ragged tail chunk in one image
    keep = torch.from_numpy(keep_np)
    qd, kd, vd, keepd = _dev(q, k, v, keep)
    ref, _ = fused_oracle(q, k, v, keep)
    o_long = rb.pack_attend_unpack(qd, kd, vd, keepd, n_hint=N, engine=rb.ENGINE_MMA_SYNC)
    o_short = rb.pack_attend_unpack(qd, kd, vd, keepd)
    qp, kp, vp, cu, dst, src = rb.pack(qd, kd, vd, keepd)
    # composed path on the fused kernel's engine (AUTO takes the warp-specialised
    # engine at n_hint > 148: equal within tolerance, not bitwise -- tested below)
    o_comp = rb.unpack(rb.attn(qp, kp, vp, cu, N, n_hint=N, engine=rb.ENGINE_MMA_SYNC), dst, B, N)
    o_auto = rb.unpack(rb.attn(qp, kp, vp, cu, N, n_hint=N), dst, B, N)
    torch.cuda.synchronize()
    assert np.array_equal(bits(o_long), bits(o_comp))
    check_attention(to_np(o_long), ref, DT[dtype], dist="peaked")
    check_attention(to_np(o_short), ref, DT[dtype], dist="peaked")
    check_attention(to_np(o_auto), ref, DT[dtype], dist="peaked")  # the warp-specialised engine's lazy rescale


@pytest.mark.parametrize("n_hint,engine", [(0, 0), (197, 0), (197, 3)])
def test_mask_rewritten_by_previous_kernel(n_hint, engine):
    """The fused kernel reads the keep row (and prefetches kept rows) BEFORE its
    PDL grid-dependency wait; only the post-wait read may reach results.  Here
    the N2 mask kernel rewrites ONE keep buffer right before every fused call
    (both PDL-launched on one stream, no host sync), alternating two hidden-
    state batches whose masks differ, so every speculative read can see the
    previous iteration's mask or a half-written one.  Every output must equal,
    bit for bit, the output computed with a synchronised mask."""
    B, N, H = 16, 197, 12
    kk = synth.kept_tokens(N, 0.7)
    xs = [synth.hidden_states(B, N, H * 64, "bf16", seed=s).to(DEV) for s in (11, 12)]
    q, k, v = _dev(*synth.activations(B, N, H, 64, "bf16", seed=11))
    ref = []
    for x in xs:
        km = rb.keep_topk_l2(x, kk)
        torch.cuda.synchronize()
        ref.append(rb.pack_attend_unpack(q, k, v, km, n_hint=n_hint, engine=engine))
        torch.cuda.synchronize()
    assert not torch.equal(rb.keep_topk_l2(xs[0], kk), rb.keep_topk_l2(xs[1], kk))
    keep = torch.empty(B, N, dtype=torch.uint8, device=DEV)
    outs = [torch.empty_like(ref[0]) for _ in range(40)]
    for i, o in enumerate(outs):
        rb.keep_topk_l2(xs[i % 2], kk, keep=keep)
        rb.pack_attend_unpack(q, k, v, keep, o=o, n_hint=n_hint, engine=engine)
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        assert np.array_equal(bits(o), bits(ref[i % 2])), f"call {i}"


@pytest.mark.parametrize("n_hint", [0, 39, 197])
def test_query_split_small_batch_bitwise_equals_unsplit(n_hint):
    """Small batches split each (image, head) problem's query slices over
    several CTAs (mma.sync engine, attn_qsplit): the output must be bitwise the
    one computed with one CTA per problem (the same images inside a batch large
    enough not to split), for the fused path and ragged_attn, with cu_seqlens."""
    B, N, H = 2, 197, 3
    q, k, v, keep = synth.make_inputs(B, N, H, 0.0, "random", "bf16", seed=77)
    keep = keep.clone()
    keep[1, 150:] = 0                              # ragged: 197 and 150 tokens
    big = 120                                      # B * H = 360 >= 2 * #SMs: no split
    rep = lambda t: torch.cat([t] * (big // B)).contiguous()  # noqa: E731
    qd, kd, vd, kp = _dev(q, k, v, keep)
    Qd, Kd, Vd, Kp = _dev(rep(q), rep(k), rep(v), rep(keep))
    MMA = rb.ENGINE_MMA_SYNC  # the query split is the mma.sync engine's
    o_small, cu_small = rb.pack_attend_unpack(qd, kd, vd, kp, want_cu=True, n_hint=n_hint, engine=MMA)
    o_big = rb.pack_attend_unpack(Qd, Kd, Vd, Kp, n_hint=n_hint, engine=MMA)
    torch.cuda.synchronize()
    assert np.array_equal(bits(o_small), bits(o_big[:B]))
    assert cu_small.cpu().tolist() == [0, 197, 347]
    ref, _ = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    check_attention(to_np(o_small), ref, torch.bfloat16)
    qp, kpk, vp, cu, _, _ = rb.pack(qd, kd, vd, kp)
    Qp, Kpk, Vp, CU, _, _ = rb.pack(Qd, Kd, Vd, Kp)
    a_small = rb.attn(qp, kpk, vp, cu, N, n_hint=n_hint, engine=MMA)
    a_big = rb.attn(Qp, Kpk, Vp, CU, N, n_hint=n_hint, engine=MMA)
    torch.cuda.synchronize()
    assert np.array_equal(bits(a_small[:347]), bits(a_big[:347]))
