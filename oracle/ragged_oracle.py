"""fp64 CPU oracle for the pack-attend-unpack path of arxiv 2604.15408.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module.
The product package (`paper_2604_15408_b200`) never imports it, and this module
imports nothing from the product package: the two share no code.  The only
common dependency is `synth` (seeded input generators, no method arithmetic).

Plain, slow, obviously correct: every function writes out the definition the
paper states, in float64 (reading R1), with numpy primitives as steps
(a matmul, an exp, a gather) and no blocking, fusion or reordering.

Passages followed (PAPER.md line numbers):
  scan       §4.1 "Index computation": per-image cumulative sums produce the
             cu_seqlens offset vector and per-token destination indices
             (P:266-269); cu_seqlens in Z^{B+1}.  Stable order:
             reading R7.
  pack       §4.1 "Vectorized copy": each kept token row is copied from the
             padded [B, S, D] tensor into packed in R^{T_total x D}
             (P:262-263).  Q, K and V are packed (reading R8).
  attention  Alg. 1: per image i and head h, with
             s = cu[i], n = cu[i+1] - s, O = softmax(Q K^T / sqrt(d)) V over the
             rows [s, s+n) (bidirectional, no mask inside a sequence).
             Alg. 1's online softmax is an exact reformulation of this plain
             softmax (FA2), so the oracle computes the plain
             definition; the tiled form is pinned against it in the tests.
  unpack     Inverse of pack: packed rows return to their padded positions,
             dropped positions hold +0.0 (reading R10; not in the paper).
  fused      pack_attend_unpack = unpack o attention o pack (BASELINE.json).

  fp8        (NEXT row N4) ragged attention over FP8 E4M3 inputs with
             per-tensor scales: the bytes are decoded by the OCP E4M3 formula
             (reading R23; not in the paper) and the plain attention above is
             applied to the dequantised values.

  prune      (NEXT row N2) Threshold-l2 keep mask: l2 norm of each token's
             hidden state, CLS + top-(k-1) (R20).
  evit       (NEXT row N2) EViT-style keep mask with a fused token (P:95-96
             "ranks tokens by CLS-attention scores and fuses pruned tokens into a
             single representative"; reading R17): head-averaged CLS logits,
             CLS + top-(k-2), the dropped rows' logit-softmax-weighted mean
             written into the first dropped position, which is marked kept.

Pins (tests/test_oracle.py, run with -m "not gpu"): SPEC worked examples,
Table 1 token counts and the T = 6,304 / 12,608 totals (P:167-179, P:202,
P:238), brute-force global ranks, torch.nonzero / flash_attn.bert_padding
library routines, torch SDPA in fp64 at 0 % pruning, scipy logsumexp, the
n = 1 and n = 2 closed forms, identical keys, rows summing to 1, permutation
equivariance, cross-image isolation, and Alg. 1's tiled online softmax.
"""
from __future__ import annotations

import numpy as np


def as_f64(x) -> np.ndarray:
    """Exact upcast of a bf16/fp16/fp32 torch tensor or numpy array to float64."""
    if hasattr(x, "detach"):
        x = x.detach().cpu().double().numpy()
    return np.asarray(x, dtype=np.float64)


def scan(keep):
    """keep [B, N] (nonzero = keep) -> (cu [B+1], dst [B*N], src [B*N]).

    cu[0] = 0, cu[b+1] = cu[b] + #kept in image b
    dst[b*N + n] = cu[b] + #{n' < n kept in image b}  if kept, else -1
    src[dst[i]] = i; entries src[r] for r >= cu[B] are -1 (capacity, unused).
    """
    keep = np.asarray(keep) != 0
    B, N = keep.shape
    cu = np.zeros(B + 1, np.int64)
    dst = np.full(B * N, -1, np.int64)
    src = np.full(B * N, -1, np.int64)
    for b in range(B):
        pos = np.flatnonzero(keep[b])          # ascending original position (R7)
        rows = cu[b] + np.arange(pos.size)
        cu[b + 1] = cu[b] + pos.size
        dst[b * N + pos] = rows
        src[rows] = b * N + pos
    return cu, dst, src


def pack(x, src, T: int) -> np.ndarray:
    """x [B, N, ...] (any dtype; bit patterns are copied) -> packed [T, ...]:
    packed[r] = x[src[r]]."""
    x = np.asarray(x)
    flat = x.reshape((x.shape[0] * x.shape[1],) + x.shape[2:])
    return flat[np.asarray(src[:T], np.int64)].copy()


def attention_one(q, k, v) -> np.ndarray:
    """One (image, head) problem of Alg. 1 in its plain form, fp64:
    S = q k^T / sqrt(d) (Alg. 1 line 10); P = softmax_rows(S) computed
    as exp(S - rowmax) / rowsum; O = P v."""
    q, k, v = as_f64(q), as_f64(k), as_f64(v)
    if q.shape[0] == 0:
        return np.zeros((0, v.shape[1]))
    d = q.shape[1]
    S = (q @ k.T) / np.sqrt(d)
    m = S.max(axis=1, keepdims=True)
    e = np.exp(S - m)
    return (e / e.sum(axis=1, keepdims=True)) @ v


def softmax_weights(q, k) -> np.ndarray:
    """The n x n softmax matrix of one (image, head) problem (for the
    rows-sum-to-one pin)."""
    q, k = as_f64(q), as_f64(k)
    S = (q @ k.T) / np.sqrt(q.shape[1])
    e = np.exp(S - S.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


def attention(qp, kp, vp, cu) -> np.ndarray:
    """Packed Q, K, V [T, H, d] + cu_seqlens [B+1] -> packed O [T, H, d].
    One problem per (image i, head h): pid -> (h = pid mod H, i = pid // H)
    (Alg. 1 lines 2-4); images with n = 0 produce no rows."""
    qp, kp, vp = as_f64(qp), as_f64(kp), as_f64(vp)
    if not (np.isfinite(qp).all() and np.isfinite(kp).all() and np.isfinite(vp).all()):
        raise ValueError("oracle: non-finite input (parity is defined on finite inputs, R14)")
    T, H, d = qp.shape
    out = np.zeros((T, H, d))
    B = len(cu) - 1
    for i in range(B):
        s, e = int(cu[i]), int(cu[i + 1])
        for h in range(H):
            out[s:e, h] = attention_one(qp[s:e, h], kp[s:e, h], vp[s:e, h])
    return out


def unpack(op, dst, B: int, N: int, fill=0) -> np.ndarray:
    """Packed O [T, ...] -> padded [B, N, ...]: O[i] = op[dst[i]] if dst[i] >= 0,
    else `fill` (+0.0 by default, reading R10)."""
    op = np.asarray(op)
    dst = np.asarray(dst, np.int64)
    out = np.full((B * N,) + op.shape[1:], fill, dtype=op.dtype)
    kept = dst >= 0
    out[kept] = op[dst[kept]]
    return out.reshape((B, N) + op.shape[1:])


def pack_attend_unpack(q, k, v, keep):
    """The whole path (BASELINE.json north_star): padded Q/K/V [B, N, H, d] +
    keep [B, N] -> (padded O [B, N, H, d] in fp64 with zero rows for dropped
    tokens, cu_seqlens)."""
    q, k, v = as_f64(q), as_f64(k), as_f64(v)
    keep = np.asarray(keep)
    B, N = keep.shape
    cu, dst, src = scan(keep)
    T = int(cu[B])
    op = attention(pack(q, src, T), pack(k, src, T), pack(v, src, T), cu)
    return unpack(op, dst, B, N, 0.0), cu


def l2_scores(x) -> np.ndarray:
    """Threshold-l2 token scores (the paper names the scorer but never
    defines it, S:312 -- DESIGN.md R20): score[b, n] = ||x[b, n, :]||_2 in fp64,
    with CLS (n = 0) set to +inf so it always survives (R6)."""
    x = as_f64(x)
    s = np.sqrt((x * x).sum(axis=2))
    s[:, 0] = np.inf
    return s


def _scores_nan_low(s):
    """NaN scores rank below every finite score (R20): at most k tokens kept."""
    s = np.array(s, dtype=np.float64)
    s[np.isnan(s)] = -np.inf
    return s


def keep_topk_l2(x, k: int) -> np.ndarray:
    """keep [B, N] uint8: CLS + the k - 1 highest-scoring other tokens of each
    image ("any supported method produces a binary keep mask"); ties
    go to the lower position (stable order, R20)."""
    if k < 1:
        raise ValueError("k must be >= 1: CLS always survives (R6)")
    s = _scores_nan_low(l2_scores(x))
    B, N = s.shape
    keep = np.zeros((B, N), np.uint8)
    for b in range(B):
        order = np.argsort(-s[b], kind="stable")
        keep[b, order[:max(0, min(k, N))]] = 1
    return keep


def evit_logits(q, k) -> np.ndarray:
    """EViT token scores (R17): the CLS query's attention logits to
    every token, averaged over heads -- logit[b, n] = (1/H) sum_h
    q[b, 0, h] . k[b, n, h] / sqrt(d), fp64."""
    q, k = as_f64(q), as_f64(k)
    B, N, H, d = k.shape
    out = np.zeros((B, N))
    for b in range(B):
        for h in range(H):
            out[b] += (k[b, :, h] @ q[b, 0, h]) / np.sqrt(d)
    return out / H


def keep_evit(q, k, v, k_keep: int):
    """EViT-style keep mask with a fused token (reading R17), per image:
    1. scores = evit_logits; CLS (n = 0) always kept;
    2. keep CLS + the max(k_keep - 2, 0) highest-scoring other tokens (ties to the
       lower position);
    3. if k_keep >= 2 and a token is dropped: the fused token = sum over dropped
       tokens j of w_j * row_j with w = softmax(scores[dropped]) (CLS-attention
       weights of the dropped tokens, normalised), for each of Q, K, V and every
       head; it is written into the first dropped position f, which is kept;
    4. k_keep >= N keeps every token (no fused token).
    Returns (keep uint8 [B, N], f int [B] (-1 = none), fused fp64 [B, 3, H, d])."""
    if k_keep < 1:
        raise ValueError("k_keep must be >= 1: CLS always survives (R6)")
    s = _scores_nan_low(evit_logits(q, k))
    qf, kf, vf = as_f64(q), as_f64(k), as_f64(v)
    B, N, H, d = kf.shape
    keep = np.zeros((B, N), np.uint8)
    f = np.full(B, -1, np.int64)
    fused = np.zeros((B, 3, H, d))
    for b in range(B):
        if k_keep >= N:
            keep[b] = 1
            continue
        others = 1 + np.argsort(-s[b, 1:], kind="stable")
        keep[b, 0] = 1
        keep[b, others[:max(k_keep - 2, 0)]] = 1
        dropped = np.flatnonzero(keep[b] == 0)
        if k_keep >= 2 and dropped.size > 0:
            e = np.exp(s[b, dropped] - s[b, dropped].max())
            w = e / e.sum()
            for t, x in enumerate((qf, kf, vf)):
                fused[b, t] = np.tensordot(w, x[b, dropped], axes=(0, 0))
            f[b] = dropped[0]
            keep[b, f[b]] = 1
    return keep, f, fused


def attention_image_head(q, k, v, keep, b: int, h: int):
    """Sampled check at full size: the output rows of image b, head h, computed
    one problem at a time from the padded inputs (same definition as
    pack_attend_unpack, restricted to one (b, h)).  Returns (kept positions,
    rows [n, d])."""
    pos = np.flatnonzero(np.asarray(keep[b]) != 0)
    qb, kb, vb = (as_f64(t[b, pos, h]) for t in (q, k, v))
    return pos, attention_one(qb, kb, vb)


def e4m3_decode(b) -> np.ndarray:
    """FP8 E4M3 (OCP "e4m3fn") bytes -> exact float64 values (reading R23):
    sign s = bit 7, exponent e = bits 6..3 (bias 7), mantissa m = bits 2..0;
    e = 0: (-1)^s * m/8 * 2^-6 (subnormal); e = 15 and m = 7: NaN; otherwise
    (-1)^s * (1 + m/8) * 2^(e-7).  No infinities; max finite 448."""
    b = np.asarray(b, dtype=np.uint8).astype(np.int64)
    s = np.where(b >> 7 == 1, -1.0, 1.0)
    e = (b >> 3) & 0xF
    m = (b & 0x7).astype(np.float64)
    val = np.where(e == 0, m / 8.0 * 2.0 ** -6, (1.0 + m / 8.0) * np.power(2.0, (e - 7).astype(np.float64)))
    val = np.where((e == 15) & (b & 0x7 == 7), np.nan, val)
    return s * val


def attention_fp8(q8, k8, v8, descale, cu) -> np.ndarray:
    """NEXT row N4: packed FP8 E4M3 q/k/v bytes (uint8 arrays [T, H, d]) with
    per-tensor descale factors (dq, dk, dv): attention() of dq*decode(q),
    dk*decode(k), dv*decode(v)."""
    dq, dk, dv = (float(x) for x in descale)
    return attention(e4m3_decode(q8) * dq, e4m3_decode(k8) * dk, e4m3_decode(v8) * dv, cu)

