"""GPU parity of the warp-specialised tcgen05 engine (csrc/attn_fa.cu,
RAGGED_ENGINE_TCGEN05_WS) for ragged_attn at head_dim 64: every tile-edge
length around the 128-row query tiles / 128-key blocks and the 256-row tile
pairs, empty images, long sequences, bf16 / fp16, peaked and heavy inputs,
against the fp64 oracle with the R2 tolerances; deterministic and isolated."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import check_attention, to_np

rb = pytest.importorskip("paper_2604_15408_b200")
pytestmark = pytest.mark.gpu
DEV = "cuda"
DT = {"bf16": torch.bfloat16, "fp16": torch.float16}
WS = 3


def _case(lengths, H, dt, seed, dist="standard"):
    lengths = np.asarray(lengths)
    B, N = len(lengths), max(1, int(lengths.max()))
    q, k, v = synth.activations(B, N, H, 64, DT[dt], seed, dist)
    keep = np.zeros((B, N), np.uint8)
    for b, n in enumerate(lengths):
        keep[b, :n] = 1
    cu, _, src = oracle.scan(keep)
    T = int(cu[-1])
    idx = torch.from_numpy(src[:T])
    pk = [t.reshape(B * N, H, 64)[idx] for t in (q, k, v)]
    cap = [torch.cat([t, torch.zeros(B * N - T, H, 64, dtype=t.dtype)]) for t in pk]
    return pk, [t.to(DEV) for t in cap], cu, N, T


def _run(cap, cu, N, **kw):
    cud = torch.from_numpy(cu.astype(np.int32)).to(DEV)
    out = rb.attn(*cap, cud, N, engine=WS, **kw)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
@pytest.mark.parametrize("lengths", [[1, 2, 17, 64, 65], [127, 128, 129, 0, 197],
                                     [255, 256, 257, 383, 384, 385], [577, 39, 1000], [513, 0, 0, 2]])
def test_ws_lengths(dt, lengths):
    pk, cap, cu, N, T = _case(lengths, 3, dt, seed=sum(lengths) % 97)
    got = _run(cap, cu, N)
    check_attention(to_np(got[:T]), oracle.attention(*pk, cu), DT[dt])


@pytest.mark.parametrize("dist", ["peaked", "heavy"])
def test_ws_distributions(dist):
    """Peaked scores exercise the lazy rescaling across 128-key blocks (rising
    maxima); heavy V the secondary bound."""
    pk, cap, cu, N, T = _case([600, 250, 131], 2, "bf16", seed=21, dist=dist)
    got = _run(cap, cu, N)
    vmax = float(pk[2].abs().max()) if dist == "heavy" else None
    check_attention(to_np(got[:T]), oracle.attention(*pk, cu), torch.bfloat16, vmax=vmax, dist=dist)


def test_ws_rising_scores_force_rescale():
    """Scores increasing block by block (key j aligned with the query more for
    larger j) make every block raise the reference max: the O-row rescale path."""
    B, n, H = 1, 700, 2
    q = torch.zeros(B, n, H, 64)
    q[..., 0] = 4.0
    k = torch.zeros(B, n, H, 64)
    k[..., 0] = torch.linspace(-3, 3, n)[None, :, None]
    v = torch.rand(B, n, H, 64) * 2 - 1
    q, k, v = (t.to(torch.bfloat16) for t in (q, k, v))
    cu = np.array([0, n])
    pk = [t.reshape(n, H, 64) for t in (q, k, v)]
    got = _run([t.to(DEV) for t in pk], cu, n)
    check_attention(to_np(got), oracle.attention(*pk, cu), torch.bfloat16)


def test_ws_matches_mma_engine_and_is_deterministic():
    pk, cap, cu, N, T = _case([197] * 16, 12, "bf16", seed=5)
    a = _run(cap, cu, N)
    b = _run(cap, cu, N)
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    ref = oracle.attention(*pk, cu)
    m = rb.attn(*cap, torch.from_numpy(cu.astype(np.int32)).to(DEV), N, engine=rb.ENGINE_MMA_SYNC)
    torch.cuda.synchronize()
    check_attention(to_np(a[:T]), ref, torch.bfloat16)
    check_attention(to_np(m[:T]), ref, torch.bfloat16)


def test_ws_isolation_and_untouched_rows():
    pk, cap, cu, N, T = _case([300, 90, 0, 140], 2, "fp16", seed=8)
    op = torch.full_like(cap[0], 7.0)
    cud = torch.from_numpy(cu.astype(np.int32)).to(DEV)
    rb.attn(*cap, cud, N, op=op, engine=WS)
    k2 = cap[1].clone()
    k2[300:390] += 1.0                                   # perturb image 1 only
    op2 = rb.attn(cap[0], k2, cap[2], cud, N, engine=WS)
    torch.cuda.synchronize()
    assert (op[T:] == 7.0).all()
    assert torch.equal(op[:300].view(torch.int16), op2[:300].view(torch.int16))
    assert torch.equal(op[390:T].view(torch.int16), op2[390:T].view(torch.int16))


@pytest.mark.parametrize("n_hint,engine", [(197, WS), (158, WS), (138, 1), (39, 1), (0, 1)])
def test_auto_engine_choice_by_n_hint(n_hint, engine):
    """AUTO at N <= 256: the warp-specialised engine when the caller expects more
    than 148 kept tokens per image (measured crossover), the mma.sync kernels
    otherwise -- the AUTO result is bitwise the chosen engine's (same n_hint)."""
    pk, cap, cu, N, T = _case([197, 150, 60, 197], 4, "bf16", seed=n_hint)
    cud = torch.from_numpy(cu.astype(np.int32)).to(DEV)
    auto = rb.attn(*cap, cud, N, engine=rb.ENGINE_AUTO, n_hint=n_hint)
    ref = rb.attn(*cap, cud, N, engine=engine, n_hint=n_hint)
    torch.cuda.synchronize()
    assert torch.equal(auto[:T].view(torch.int16), ref[:T].view(torch.int16))
    check_attention(to_np(auto[:T]), oracle.attention(*pk, cu), torch.bfloat16)


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
@pytest.mark.parametrize("B,N,H,p,method", [(3, 197, 2, 0.0, "all"), (4, 197, 3, 0.5, "l2"), (5, 256, 2, 0.2, "random"),
                                            (2, 33, 4, 0.5, "ats"), (6, 197, 12, 0.8, "l2"), (2, 1, 2, 0.0, "all"),
                                            (40, 197, 6, 0.3, "dynamicvit")])
def test_ws_fused_pack_attend_unpack(dt, B, N, H, p, method):
    """ragged_pack_attend_unpack on the warp-specialised engine (TMA tile::gather4
    of the kept rows of the padded q/k/v, the packed engine's attention, O rows
    stored at their padded positions, +0.0 rows written by the rows warps):
    within the R2 tolerance of the fp64 oracle, cu_seqlens bit-exact, every
    dropped row +0.0, an empty image all +0.0, run-to-run deterministic."""
    q, k, v, keep = synth.make_inputs(B, N, H, p, method, dt, seed=B * N + H)
    keep = keep.clone()
    if B > 2:
        keep[1] = 0
    qd, kd, vd, kpd = (t.to(DEV) for t in (q, k, v, keep))
    o1 = torch.full((B, N, H, 64), 7.0, dtype=DT[dt], device=DEV)
    cu = torch.full((B + 1,), -5, dtype=torch.int32, device=DEV)
    rb.pack_attend_unpack(qd, kd, vd, kpd, o=o1, cu=cu, engine=WS)
    o2 = rb.pack_attend_unpack(qd, kd, vd, kpd, engine=WS)
    torch.cuda.synchronize()
    ref, rcu = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    assert cu.cpu().tolist() == rcu.tolist()
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
    check_attention(to_np(o1), ref, DT[dt])
    kb = keep.numpy().astype(bool)
    assert (o1.cpu().view(torch.int16).numpy()[~kb] == 0).all()


def test_ws_fused_qkv_layout():
    """One fused [B, N, 3, H, d] qkv buffer (token stride 3 H d) through the gather4 path."""
    B, N, H = 4, 197, 3
    q, k, v, keep = synth.make_inputs(B, N, H, 0.3, "l2", "bf16", seed=9)
    qkv = torch.stack([q, k, v], dim=2).to(DEV)
    o = rb.pack_attend_unpack(qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2], keep.to(DEV), engine=WS)
    torch.cuda.synchronize()
    ref, _ = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    check_attention(to_np(o), ref, torch.bfloat16)


@pytest.mark.parametrize("B,n_hint,engine", [(32, 197, WS), (32, 188, WS), (32, 187, 1), (32, 39, 1), (6, 197, 1)])
def test_fused_auto_engine_choice(B, n_hint, engine):
    """AUTO for the fused call: the warp-specialised engine only for nearly
    unpruned images (n_hint >= 188) and at least two (image, head) problems per
    SM, else the one-stage kernels; bitwise the chosen engine's result."""
    N, H = 197, 12
    q, k, v, keep = (t.to(DEV) for t in synth.make_inputs(B, N, H, 0.0, "all", "bf16", seed=n_hint))
    auto = rb.pack_attend_unpack(q, k, v, keep, n_hint=n_hint)
    ref = rb.pack_attend_unpack(q, k, v, keep, n_hint=n_hint, engine=engine)
    torch.cuda.synchronize()
    assert torch.equal(auto.view(torch.int16), ref.view(torch.int16))
