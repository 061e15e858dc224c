"""GPU parity of NEXT row N4 (csrc/attn_general.cu): ragged_attn for head dims
d in {32, 64, 80, 128} and sequences longer than the one-stage cap (N > 256),
against the fp64 oracle (oracle.attention, which is shape-generic).  Same
tolerance as the DeiT path (R2): max-abs <= 2e-3 (bf16) / 5e-4 (fp16) with
V ~ U(-1, 1), plus the secondary bound ulp(|ref|) + 2^-12 max|V|."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import TOL, check_attention, to_np

rb = pytest.importorskip("paper_2604_15408_b200")
pytestmark = pytest.mark.gpu
DEV = "cuda"
DT = {"bf16": torch.bfloat16, "fp16": torch.float16}


def _packed_case(lengths, H, d, dt, seed, dist="standard"):
    lengths = np.asarray(lengths)
    B, N = len(lengths), max(1, int(lengths.max()))
    q, k, v = synth.activations(B, N, H, d, DT[dt], seed, dist)
    keep = np.zeros((B, N), np.uint8)
    for b, n in enumerate(lengths):
        keep[b, :n] = 1
    cu, _, src = oracle.scan(keep)
    T = int(cu[-1])
    flat = lambda t: t.reshape(B * N, H, d)[torch.from_numpy(src[:T])]  # noqa: E731
    qp, kp, vp = (flat(t) for t in (q, k, v))
    return qp, kp, vp, cu, N, T


def _cap(t, rows):
    """Pad a packed [T, H, d] tensor to `rows` (the binding requires the B*N-row
    capacity that ragged_pack produces)."""
    if t.shape[0] >= rows:
        return t
    pad = torch.zeros((rows - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    return torch.cat([t, pad])


def attn_cap(qp, kp, vp, cu, N, **kw):
    rows = (cu.numel() - 1) * N
    T = qp.shape[0]
    return rb.attn(_cap(qp, rows), _cap(kp, rows), _cap(vp, rows), cu, N, **kw)[:T]


def attn_fp8_cap(qp, kp, vp, cu, N, *a, **kw):
    rows = (cu.numel() - 1) * N
    T = qp.shape[0]
    pad = lambda t: _cap(t.view(torch.uint8), rows).view(t.dtype)  # noqa: E731
    return rb.attn_fp8(pad(qp), pad(kp), pad(vp), cu, N, *a, **kw)[:T]


@pytest.mark.parametrize("d", [32, 64, 80, 128])
@pytest.mark.parametrize("dt", ["bf16", "fp16"])
def test_general_head_dims(d, dt):
    lengths = [197, 1, 0, 63, 64, 65, 130, 39, 256]
    H = 3
    qp, kp, vp, cu, N, T = _packed_case(lengths, H, d, dt, seed=d)
    cud = torch.from_numpy(cu.astype(np.int32)).to(DEV)
    got = attn_cap(qp.to(DEV), kp.to(DEV), vp.to(DEV), cud, N)
    torch.cuda.synchronize()
    ref = oracle.attention(qp, kp, vp, cu)
    check_attention(to_np(got[:T]), ref, DT[dt])


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
def test_general_long_sequences(dt):
    """N > 256: Alg. 1's K/V streaming (ViT-L/16 @ 384: 577 tokens; 1000; a
    ragged mix)."""
    lengths = [577, 1000, 300, 257, 5]
    qp, kp, vp, cu, N, T = _packed_case(lengths, 2, 64, dt, seed=7)
    got = attn_cap(qp.to(DEV), kp.to(DEV), vp.to(DEV), torch.from_numpy(cu.astype(np.int32)).to(DEV), N)
    torch.cuda.synchronize()
    check_attention(to_np(got[:T]), oracle.attention(qp, kp, vp, cu), DT[dt])


@pytest.mark.parametrize("dist", ["peaked", "heavy"])
def test_general_distributions(dist):
    lengths = [400, 77, 129]
    qp, kp, vp, cu, N, T = _packed_case(lengths, 2, 128, "bf16", seed=9, dist=dist)
    got = attn_cap(qp.to(DEV), kp.to(DEV), vp.to(DEV), torch.from_numpy(cu.astype(np.int32)).to(DEV), N)
    torch.cuda.synchronize()
    vmax = float(vp.abs().max()) if dist == "heavy" else None
    check_attention(to_np(got[:T]), oracle.attention(qp, kp, vp, cu), torch.bfloat16, vmax=vmax, dist=dist)


def test_general_strided_qkv_and_untouched_rows():
    """Packed qkv buffer [cap, 3, H, d] (row stride 3*H*d), d = 80; output rows
    past cu[B] keep their contents."""
    lengths = [300, 45, 0, 260]
    H, d = 2, 80
    qp, kp, vp, cu, N, T = _packed_case(lengths, H, d, "bf16", seed=11)
    cap = max(T + 37, len(lengths) * N)
    qkv = torch.zeros(cap, 3, H, d, dtype=torch.bfloat16)
    qkv[:T, 0], qkv[:T, 1], qkv[:T, 2] = qp, kp, vp
    qkv = qkv.to(DEV)
    op = torch.full((cap, H, d), 7.0, dtype=torch.bfloat16, device=DEV)
    rb.attn(qkv[:, 0], qkv[:, 1], qkv[:, 2], torch.from_numpy(cu.astype(np.int32)).to(DEV), N, op=op)
    torch.cuda.synchronize()
    check_attention(to_np(op[:T]), oracle.attention(qp, kp, vp, cu), torch.bfloat16)
    assert (op[T:] == 7.0).all()


def test_general_deterministic_and_isolated():
    lengths = [333, 90]
    qp, kp, vp, cu, N, T = _packed_case(lengths, 2, 128, "bf16", seed=13)
    cud = torch.from_numpy(cu.astype(np.int32)).to(DEV)
    a = attn_cap(qp.to(DEV), kp.to(DEV), vp.to(DEV), cud, N)
    b = attn_cap(qp.to(DEV), kp.to(DEV), vp.to(DEV), cud, N)
    kp2 = kp.clone()
    kp2[333:] += 1.0                       # perturb image 1 only
    c = attn_cap(qp.to(DEV), kp2.to(DEV), vp.to(DEV), cud, N)
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    assert torch.equal(a[:333].view(torch.int16), c[:333].view(torch.int16))


def _quant_e4m3(x):
    """Per-tensor FP8 E4M3 quantisation with scale amax / 448 (an fp32 value)."""
    s = float(np.float32(float(x.abs().max()) / 448.0))
    return (x.float() / s).to(torch.float8_e4m3fn), s


@pytest.mark.parametrize("d", [32, 64, 80, 128])
@pytest.mark.parametrize("out", ["bf16", "fp16"])
def test_general_fp8_inputs(d, out):
    """NEXT row N4, fp8 inputs: packed E4M3 q/k/v + per-tensor descales
    (ragged_attn_fp8) vs the oracle on the dequantised values (R23); ragged
    lengths incl. empty, 1, tile edges and N > 256; output bf16 / fp16 within
    the output type's tolerance."""
    lengths = [197, 1, 0, 63, 64, 65, 130, 39, 300]
    H = 3
    qp, kp, vp, cu, N, T = _packed_case(lengths, H, d, "fp16", seed=100 + d)
    (q8, sq), (k8, sk), (v8, sv) = (_quant_e4m3(t) for t in (qp, kp, vp))
    cud = torch.from_numpy(cu.astype(np.int32)).to(DEV)
    got = attn_fp8_cap(q8.to(DEV), k8.to(DEV), v8.to(DEV), cud, N, (sq, sk, sv), out_dtype=DT[out])
    torch.cuda.synchronize()
    u8 = lambda t: t.view(torch.uint8).numpy()  # noqa: E731
    ref = oracle.attention_fp8(u8(q8), u8(k8), u8(v8), (sq, sk, sv), cu)
    check_attention(to_np(got[:T]), ref, DT[out])


def test_general_fp8_deit_shape_and_peaked():
    """DeiT-B packing at 80 % (39 tokens/image, H = 12, d = 64) with peaked
    scores (Q, K x 3 before quantisation)."""
    lengths = [39] * 32
    qp, kp, vp, cu, N, T = _packed_case(lengths, 12, 64, "bf16", seed=5, dist="peaked")
    (q8, sq), (k8, sk), (v8, sv) = (_quant_e4m3(t) for t in (qp, kp, vp))
    got = attn_fp8_cap(q8.to(DEV), k8.to(DEV), v8.to(DEV), torch.from_numpy(cu.astype(np.int32)).to(DEV), 197,
                      (sq, sk, sv))
    torch.cuda.synchronize()
    u8 = lambda t: t.view(torch.uint8).numpy()  # noqa: E731
    check_attention(to_np(got[:T]), oracle.attention_fp8(u8(q8), u8(k8), u8(v8), (sq, sk, sv), cu),
                    torch.bfloat16)
