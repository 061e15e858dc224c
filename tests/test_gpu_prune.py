"""GPU parity for NEXT row N2's EViT keep mask (ragged_keep_evit, R17) against
the fp64 oracle: the kept set is exact wherever the decision is unique (the
score gap at the threshold is well above fp32 rounding), otherwise it must be a
valid top-k; the fused token (written in place into q/k/v at the first dropped
position) is within one output ulp + fp32 accumulation error of the oracle;
every other q/k/v byte is untouched; the result drives the fused path."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import bits, check_attention, to_np

rb = pytest.importorskip("paper_2604_15408_b200")
pytestmark = pytest.mark.gpu
DEV = "cuda"
DT = {"bf16": torch.bfloat16, "fp16": torch.float16}


def _check_evit(q, k, v, kk, keep_gpu, q2, k2, v2):
    """q, k, v: host inputs; q2/k2/v2: device results (in place)."""
    want, f, fused = oracle.keep_evit(q, k, v, kk)
    s = oracle.evit_logits(q, k)
    B, N = want.shape
    qkv_in = (q, k, v)
    qkv_out = [t.cpu() for t in (q2, k2, v2)]
    exact = 0
    for b in range(B):
        got = keep_gpu[b]
        assert got.sum() == min(kk, N) and got[0] == 1, b
        if np.array_equal(got, want[b]):
            exact += 1
            if f[b] >= 0:
                for t in range(3):
                    g = qkv_out[t][b, f[b]].double().numpy()
                    ref = fused[b, t]
                    scale = np.abs(qkv_in[t][b].double().numpy()).max()
                    ulp = np.abs(ref) * 2.0 ** (-7 if qkv_in[t].dtype == torch.bfloat16 else -10)
                    assert np.all(np.abs(g - ref) <= ulp + 2.0 ** -16 * scale), (b, t)
            # every other row untouched (bitwise)
            for t in range(3):
                rows = [n for n in range(N) if n != f[b]]
                assert np.array_equal(bits(qkv_out[t][b, rows]), bits(qkv_in[t][b, rows])), (b, t)
            continue
        others = np.sort(s[b, 1:])[::-1]
        j = kk - 2
        gap = abs(others[j - 1] - others[j]) if 0 < j < others.size else np.inf
        assert gap < 1e-5 * max(1.0, np.abs(others).max()), f"image {b}: masks differ, gap {gap:.2e}"
    return exact


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("B,N,H,p", [(64, 197, 12, 0.7), (4, 197, 3, 0.5), (7, 33, 2, 0.3), (3, 256, 6, 0.9),
                                     (2, 5, 1, 0.5), (5, 197, 12, 0.99)])
def test_keep_evit_matches_oracle(dtype, B, N, H, p):
    q, k, v = synth.activations(B, N, H, 64, dtype, seed=41)
    kk = max(1, synth.kept_tokens(N, p))
    qd, kd, vd = (t.to(DEV) for t in (q, k, v))
    keep = rb.keep_evit(qd, kd, vd, kk)
    torch.cuda.synchronize()
    assert _check_evit(q, k, v, kk, keep.cpu().numpy(), qd, kd, vd) >= B - 1


@pytest.mark.parametrize("kk", [1, 2, 3, 196, 197, 300])
def test_keep_evit_k_edges(kk):
    """k = 1: CLS only, no fused token; k = 2: CLS + fused token; k = N - 1: two
    dropped tokens fused into one; k >= N: all kept, q/k/v untouched."""
    B, N, H = 3, 197, 4
    q, k, v = synth.activations(B, N, H, 64, "bf16", seed=42)
    qd, kd, vd = (t.to(DEV) for t in (q, k, v))
    keep = rb.keep_evit(qd, kd, vd, kk).cpu().numpy()
    torch.cuda.synchronize()
    _check_evit(q, k, v, kk, keep, qd, kd, vd)
    if kk >= N:
        assert keep.sum() == B * N
        for a, b in ((q, qd), (k, kd), (v, vd)):
            assert np.array_equal(bits(a), bits(b.cpu()))


def test_keep_evit_rejects_bad_k_and_is_deterministic():
    B, N, H = 6, 197, 12
    q, k, v = synth.activations(B, N, H, 64, "bf16", seed=43)
    with pytest.raises(rb.RaggedError):
        rb.keep_evit(*(t.to(DEV) for t in (q, k, v)), 0)
    outs = []
    for _ in range(3):
        qd, kd, vd = (t.to(DEV) for t in (q, k, v))
        keep = rb.keep_evit(qd, kd, vd, 59)
        torch.cuda.synchronize()
        outs.append((keep.cpu().numpy(), bits(qd.cpu()), bits(kd.cpu()), bits(vd.cpu())))
    for o in outs[1:]:
        assert all(np.array_equal(a, b) for a, b in zip(o, outs[0]))


def test_keep_evit_fused_qkv_layout_then_fused_path():
    """EViT on one fused [B, N, 3, H, d] qkv buffer (ld = 3*H*d), then the fused
    pack-attend-unpack on the mask and the modified rows, PDL-chained with no
    host sync: equals the oracle end to end (keep_evit -> pack_attend_unpack)."""
    B, N, H = 8, 197, 12
    kk = synth.kept_tokens(N, 0.7)
    q, k, v = synth.activations(B, N, H, 64, "bf16", seed=44)
    qkv = torch.stack([q, k, v], dim=2).to(DEV)                    # [B, N, 3, H, d]
    qd, kd, vd = qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2]
    keep = rb.keep_evit(qd, kd, vd, kk)
    o = rb.pack_attend_unpack(qd, kd, vd, keep, n_hint=kk)
    torch.cuda.synchronize()
    km = keep.cpu().numpy()
    _check_evit(q, k, v, kk, km, qd, kd, vd)
    ref, _ = oracle.pack_attend_unpack(qd.cpu(), kd.cpu(), vd.cpu(), km)
    check_attention(to_np(o), ref, torch.bfloat16)


# ------------------------- N2 fused ahead of the scan (Threshold-l2) ----

def _l2_mask_ok(x, k, got):
    """Exact where the threshold gap exceeds fp32 rounding; else a valid top-k."""
    want = oracle.keep_topk_l2(x, k)
    s = oracle.l2_scores(x)
    for b in range(want.shape[0]):
        if np.array_equal(got[b], want[b]):
            continue
        srt = np.sort(s[b])[::-1]
        kk = min(k, s.shape[1])
        gap = (srt[kk - 1] - srt[kk]) / srt[kk] if kk < s.shape[1] else np.inf
        assert gap < 1e-5, f"image {b}: masks differ although the threshold gap is {gap:.2e}"
        assert got[b].sum() == want[b].sum() and got[b][0] == 1


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("B,N,H,p", [(32, 197, 12, 0.8), (4, 197, 3, 0.5), (7, 33, 6, 0.3), (3, 256, 16, 0.9),
                                     (5, 197, 12, 0.0), (2, 1, 4, 0.0), (6, 100, 12, 0.5),
                                     (3, 150, 10, 0.6), (2, 197, 14, 0.8), (2, 64, 9, 0.5), (2, 256, 16, 0.0)])
def test_prune_l2_fused_matches_oracle(dtype, B, N, H, p):
    """Mask computed inside the fused launch == ragged_keep_topk_l2's definition
    (oracle), output == oracle pack-attend-unpack on that mask, cu = b*min(k,N);
    and bit-identical to the two-launch path (mask kernel -> fused kernel) on the
    same mask (same attention kernel variant)."""
    kk = max(1, synth.kept_tokens(N, p))
    x = synth.hidden_states(B, N, H * 64, dtype, seed=51)
    q, k, v = synth.activations(B, N, H, 64, dtype, seed=52)
    xd, qd, kd, vd = (t.to(DEV) for t in (x, q, k, v))
    keep = torch.empty(B, N, dtype=torch.uint8, device=DEV)
    cu = torch.empty(B + 1, dtype=torch.int32, device=DEV)
    o = rb.prune_l2_pack_attend_unpack(xd, qd, kd, vd, kk, keep=keep, cu=cu)
    torch.cuda.synchronize()
    km = keep.cpu().numpy()
    _l2_mask_ok(x, kk, km)
    assert cu.cpu().tolist() == [b * min(kk, N) for b in range(B + 1)]
    ref, _ = oracle.pack_attend_unpack(q, k, v, km)
    check_attention(to_np(o), ref, DT[dtype])
    # the prune-fused kernel is the mma.sync engine (AUTO would take the WS engine at n_hint >= 188)
    o2 = rb.pack_attend_unpack(qd, kd, vd, keep, n_hint=min(kk, N), engine=rb.ENGINE_MMA_SYNC)
    torch.cuda.synchronize()
    assert np.array_equal(bits(o), bits(o2))


def test_prune_l2_fused_pipelined_masks_change():
    """40 PDL-chained fused-prune calls on one stream alternating two hidden-state
    batches (different masks) into ONE output buffer set: every call equals the
    synchronised result bit for bit (nothing read before the grid-dependency
    wait reaches a result)."""
    B, N, H = 16, 197, 12
    kk = synth.kept_tokens(N, 0.7)
    xs = [synth.hidden_states(B, N, H * 64, "bf16", seed=s).to(DEV) for s in (61, 62)]
    q, k, v = (t.to(DEV) for t in synth.activations(B, N, H, 64, "bf16", seed=63))
    ref = []
    for x in xs:
        ref.append(rb.prune_l2_pack_attend_unpack(x, q, k, v, kk))
        torch.cuda.synchronize()
    assert not torch.equal(ref[0], ref[1])
    outs = [torch.empty_like(ref[0]) for _ in range(40)]
    keep = torch.empty(B, N, dtype=torch.uint8, device=DEV)
    for i, o in enumerate(outs):
        rb.prune_l2_pack_attend_unpack(xs[i % 2], q, k, v, kk, o=o, keep=keep)
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        assert np.array_equal(bits(o), bits(ref[i % 2])), f"call {i}"


def test_prune_l2_fused_validation():
    q = torch.zeros(2, 9, 17, 64, dtype=torch.bfloat16, device=DEV)
    x = torch.zeros(2, 9, 17 * 64, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(rb.RaggedError):
        rb.prune_l2_pack_attend_unpack(x, q, q, q, 3)          # H = 17 > 16
    q = q[:, :, :4].contiguous()
    x = x[:, :, :256].contiguous()
    with pytest.raises(rb.RaggedError):
        rb.prune_l2_pack_attend_unpack(x, q, q, q, 0)          # k < 1
