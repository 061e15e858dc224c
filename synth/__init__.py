"""Seeded synthetic inputs for the pack-attend-unpack path (arxiv 2604.15408).

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NO arithmetic of the method itself (no scan, pack, attention or
unpack): it only draws activations Q/K/V and keep masks, with the shapes and
structure of the paper's workloads.  Everything is deterministic in `seed`, and
per-image seeding makes any contiguous image range (a rank's shard) byte-equal
to the same slice of the full batch.

Paper anchors (PAPER.md line numbers):
  * DeiT-Ti/S/B shapes: H = 3/6/12 heads, d = 64, S = 197 tokens incl. CLS
    (Table 4).
  * Tokens kept per image: 197 / 99 / 39 at 0 / 50 / 80 % pruning (Table 1,
    P:167-179) -> `kept_tokens` (reading R5).
  * Mask producers: Threshold-l2, DynamicViT, EViT, ATS (P:93-98, P:140-141,
    P:421-424); the path is agnostic to the method.  The learned
    networks need trained weights, so these are synthetic stand-ins with the
    same structure (uniform k, spatially clustered, fused token, per-image k).
"""
from __future__ import annotations

import math

import numpy as np
import torch

N_DEIT = 197          # 196 patches + CLS
HEAD_DIM = 64         # B_D = d = 64

PRESETS = {
    "deit_tiny": {"H": 3, "D": 192, "MLP": 768},
    "deit_small": {"H": 6, "D": 384, "MLP": 1536},
    "deit_base": {"H": 12, "D": 768, "MLP": 3072},
}

DTYPES = {"bf16": torch.bfloat16, "fp16": torch.float16}


def kept_tokens(N: int, p: float) -> int:
    """Tokens kept per image at pruning ratio p, CLS included.

    k(p) = N - round_half_even(p * N).  Reproduces Table 1's 197/99/39 at
    p = 0/0.5/0.8; reading R5 (SPEC's rule gives 41).
    """
    if not (0.0 <= p < 1.0):
        raise ValueError("pruning ratio must be in [0, 1)")
    return max(1, N - int(round(p * N)))   # Python round() is half-to-even


def _img_rng(seed: int, b: int, stream: int) -> np.random.Generator:
    return np.random.default_rng([int(seed), int(stream), int(b)])


def _img_gen(seed: int, b: int, stream: int) -> torch.Generator:
    g = torch.Generator()
    g.manual_seed((int(seed) * 1_000_003 + int(stream) * 7_919 + int(b)) & 0x7FFFFFFFFFFF)
    return g


def activations(B: int, N: int, H: int, d: int = HEAD_DIM, dtype=torch.bfloat16,
                seed: int = 0, dist: str = "standard", image_offset: int = 0):
    """Padded Q, K, V of shape [B, N, H, d] (token-major) on the CPU.

    Drawn in fp32 from per-image generators, rounded once (RNE) to `dtype`.
      standard: Q, K ~ N(0, 1); V ~ U(-1, 1)   (|O| < 1 by convexity)
      peaked:   Q, K ~ 3 N(0, 1); V ~ U(-1, 1) (score std ~9, stresses max)
      heavy:    Q, K ~ N(0, 1); V ~ 3 t_3      (secondary tolerance only)
    """
    if isinstance(dtype, str):
        dtype = DTYPES[dtype]
    q = torch.empty(B, N, H, d, dtype=dtype)
    k = torch.empty_like(q)
    v = torch.empty_like(q)
    qk_scale = 3.0 if dist == "peaked" else 1.0
    for b in range(B):
        g = _img_gen(seed, image_offset + b, 1)
        shp = (N, H, d)
        q[b] = (torch.randn(shp, generator=g) * qk_scale).to(dtype)
        k[b] = (torch.randn(shp, generator=g) * qk_scale).to(dtype)
        if dist == "heavy":
            z = torch.randn(shp, generator=g)
            c = torch.randn((3,) + shp, generator=g).pow(2).sum(0) / 3.0
            v[b] = (3.0 * z / c.sqrt()).to(dtype)
        elif dist in ("standard", "peaked"):
            v[b] = (torch.rand(shp, generator=g) * 2.0 - 1.0).to(dtype)
        else:
            raise ValueError(f"unknown dist {dist!r}")
    return q, k, v


def hidden_states(B: int, N: int, D: int, dtype=torch.bfloat16, seed: int = 0,
                  image_offset: int = 0) -> torch.Tensor:
    """Synthetic hidden states x [B, N, D] at the prune point (after layer 4,
    P:361-362): per-token LogNormal(0, 0.5) scale times N(0, I_D), rounded once
    to `dtype` -- the heavy-tailed token norms Threshold-l2 ranks."""
    if isinstance(dtype, str):
        dtype = DTYPES[dtype]
    x = torch.empty(B, N, D, dtype=dtype)
    for b in range(B):
        g = _img_gen(seed, image_offset + b, 2)
        scale = torch.exp(0.5 * torch.randn(N, 1, generator=g))
        x[b] = (scale * torch.randn(N, D, generator=g)).to(dtype)
    return x


VIT_PARAMS = ("ln1_w", "ln1_b", "w_qkv", "b_qkv", "w_proj", "b_proj",
              "ln2_w", "ln2_b", "w_fc1", "b_fc1", "w_fc2", "b_fc2")


def vit_weights(D: int, MLP: int, dtype=torch.bfloat16, seed: int = 0) -> dict:
    """Random-init weights of one pre-norm ViT block (NEXT row N1; DeiT layout:
    qkv [3D, D] with output order (q|k|v, head, d), proj [D, D], fc1 [MLP, D],
    fc2 [D, MLP], LayerNorm weight/bias [D]); there are no trained weights in
    this build.  Linear weights ~ N(0, 0.02^2) (timm's trunc-normal scale),
    biases ~ N(0, 0.02^2) (nonzero so a dropped bias is visible), LayerNorm
    weight ~ 1 + N(0, 0.1^2), bias ~ N(0, 0.05^2).  Rounded once to `dtype`."""
    if isinstance(dtype, str):
        dtype = DTYPES[dtype]
    g = torch.Generator().manual_seed(0x5EED0000 + seed)
    shapes = {"ln1_w": (D,), "ln1_b": (D,), "w_qkv": (3 * D, D), "b_qkv": (3 * D,),
              "w_proj": (D, D), "b_proj": (D,), "ln2_w": (D,), "ln2_b": (D,),
              "w_fc1": (MLP, D), "b_fc1": (MLP,), "w_fc2": (D, MLP), "b_fc2": (D,)}
    out = {}
    for name in VIT_PARAMS:
        r = torch.randn(shapes[name], generator=g)
        if name in ("ln1_w", "ln2_w"):
            t = 1.0 + 0.1 * r
        elif name in ("ln1_b", "ln2_b"):
            t = 0.05 * r
        else:
            t = 0.02 * r
        out[name] = t.to(dtype)
    return out


def packed_rows(T: int, D: int, dtype=torch.bfloat16, seed: int = 0) -> torch.Tensor:
    """Packed hidden rows x [T, D] for the N1 block: N(0, 1) per element with a
    per-row LogNormal(0, 0.5) scale (the prune-point statistics of
    hidden_states), rounded once to `dtype`."""
    if isinstance(dtype, str):
        dtype = DTYPES[dtype]
    g = torch.Generator().manual_seed(0x9ACC0000 + seed)
    scale = torch.exp(0.5 * torch.randn(T, 1, generator=g))
    return (scale * torch.randn(T, D, generator=g)).to(dtype)


# --------------------------------------------------------------------------
# keep-mask generators: uint8 [B, N], nonzero = keep, CLS (position 0) kept.
# --------------------------------------------------------------------------

def _topk_keep(scores: np.ndarray, k: int) -> np.ndarray:
    """Keep CLS + the top-(k-1) non-CLS positions; ties go to the lower index."""
    N = scores.shape[0]
    keep = np.zeros(N, np.uint8)
    keep[0] = 1
    if k > 1:
        order = np.argsort(-scores[1:], kind="stable") + 1
        keep[order[: k - 1]] = 1
    return keep


def mask_all(B: int, N: int) -> np.ndarray:
    return np.ones((B, N), np.uint8)


def mask_threshold_l2(B: int, N: int, k: int, seed: int = 1000, image_offset: int = 0,
                      D: int = 768) -> np.ndarray:
    """Threshold-l2: score = ||x_{b,n}||_2 of a synthetic hidden
    state whose per-token scale is LogNormal(0, 0.5); keep CLS + top-(k-1).
    ||z|| for z ~ N(0, I_D) is drawn directly as sqrt(chi2_D)."""
    out = np.empty((B, N), np.uint8)
    for b in range(B):
        r = _img_rng(seed, image_offset + b, 11)
        scale = np.exp(0.5 * r.standard_normal(N))
        s = scale * np.sqrt(r.chisquare(D, N))
        out[b] = _topk_keep(s, k)
    return out


def mask_random(B: int, N: int, k: int, seed: int = 1000, image_offset: int = 0) -> np.ndarray:
    out = np.empty((B, N), np.uint8)
    for b in range(B):
        r = _img_rng(seed, image_offset + b, 12)
        out[b] = _topk_keep(r.random(N), k)
    return out


def _grid_xy(N: int):
    g = max(1, int(math.ceil(math.sqrt(max(N - 1, 1)))))
    idx = np.arange(N - 1)
    return (idx % g).astype(np.float64), (idx // g).astype(np.float64), g


def mask_dynamicvit(B: int, N: int, k: int, seed: int = 1000, image_offset: int = 0) -> np.ndarray:
    """DynamicViT-style: sigmoid(random linear head + smooth spatial
    field on the 14x14 patch grid), top-(k-1) -> spatially clustered keeps."""
    out = np.empty((B, N), np.uint8)
    x, y, g = _grid_xy(N)
    for b in range(B):
        r = _img_rng(seed, image_offset + b, 13)
        field = np.zeros(N - 1)
        for _ in range(3):
            cx, cy = r.uniform(0, g, 2)
            w = r.uniform(1.0, 3.0)
            field += r.uniform(1.0, 3.0) * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * w * w))
        logits = np.concatenate([[np.inf], 0.5 * r.standard_normal(N - 1) + field])
        s = 1.0 / (1.0 + np.exp(-logits))
        s[0] = np.inf
        out[b] = _topk_keep(s, k)
    return out


def mask_ats(B: int, N: int, k_target: int, seed: int = 1000, image_offset: int = 0,
             return_samples: bool = False):
    """ATS-style adaptive sampling (reading R16): per-image significance
    s_j = exp(tau_b g_j); M evenly spaced inverse-CDF samples over the non-CLS
    tokens, de-duplicated -> variable k_b per image.  M is calibrated by
    bisection so the batch-mean kept count is within one token of k_target."""
    sig = []
    for b in range(B):
        r = _img_rng(seed, image_offset + b, 14)
        tau = r.uniform(0.5, 2.5)
        sig.append(np.exp(tau * r.standard_normal(N - 1)))

    def build(M: int):
        out = np.zeros((B, N), np.uint8)
        out[:, 0] = 1
        u = (np.arange(M) + 0.5) / M
        for b in range(B):
            cdf = np.cumsum(sig[b])
            cdf /= cdf[-1]
            j = np.minimum(np.searchsorted(cdf, u, side="left"), N - 2)
            out[b, 1 + np.unique(j)] = 1
        return out

    if k_target >= N:
        m = mask_all(B, N)
        return (m, N) if return_samples else m
    lo, hi = 0, 64 * N          # smallest M with mean k_b >= k_target - 1/2
    while lo < hi:
        mid = (lo + hi) // 2
        if build(mid).sum(1).mean() < k_target - 0.5:
            lo = mid + 1
        else:
            hi = mid
    best = build(lo)
    return (best, lo) if return_samples else best


def mask_evit(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, k_keep: int):
    """EViT-style (reading R17): keep CLS + top-(k-2) tokens by
    head-averaged CLS logit, and write one fused token into the first dropped
    position (its Q/K/V = the CLS-weight-normalised mean of the dropped rows),
    marked kept.  Returns (mask, q', k', v') with q'/k'/v' new tensors."""
    B, N, H, d = q.shape
    q2, k2, v2 = q.clone(), k.clone(), v.clone()
    out = np.zeros((B, N), np.uint8)
    for b in range(B):
        qc = q[b, 0].double().numpy()                  # [H, d]
        kb = k[b].double().numpy()                     # [N, H, d]
        logit = np.einsum("hd,nhd->n", qc, kb) / (H * math.sqrt(d))
        if k_keep >= N:
            out[b] = 1
            continue
        keep = _topk_keep(np.concatenate([[np.inf], logit[1:]]), max(k_keep - 1, 1))
        dropped = np.flatnonzero(keep == 0)
        if k_keep >= 2 and dropped.size > 0:
            w = np.exp(logit[dropped] - logit[dropped].max())
            w /= w.sum()
            j = int(dropped[0])
            for src, dst in ((q, q2), (k, k2), (v, v2)):
                rows = src[b, dropped].double().numpy()            # [m, H, d]
                dst[b, j] = torch.from_numpy(np.einsum("m,mhd->hd", w, rows)).to(src.dtype)
            keep[j] = 1
        out[b] = keep
    return out, q2, k2, v2


MASK_METHODS = ("l2", "dynamicvit", "evit", "ats", "random", "all")


def make_inputs(B: int, N: int, H: int, p: float, method: str = "l2", dtype="bf16",
                seed: int = 0, dist: str = "standard", image_offset: int = 0, d: int = HEAD_DIM):
    """(q, k, v, keep) for one workload cell.  Masks use seed + 1000."""
    q, k, v = activations(B, N, H, d, dtype, seed, dist, image_offset)
    kk = kept_tokens(N, p)
    ms = seed + 1000
    if method == "l2":
        keep = mask_threshold_l2(B, N, kk, ms, image_offset, D=H * d)
    elif method == "dynamicvit":
        keep = mask_dynamicvit(B, N, kk, ms, image_offset)
    elif method == "evit":
        keep, q, k, v = mask_evit(q, k, v, kk)
    elif method == "ats":
        keep = mask_ats(B, N, kk, ms, image_offset)
    elif method == "random":
        keep = mask_random(B, N, kk, ms, image_offset)
    elif method == "all":
        keep = mask_all(B, N)
    else:
        raise ValueError(f"unknown mask method {method!r}")
    return q, k, v, torch.from_numpy(keep)


# The five BASELINE.json configs as concrete workloads.
CONFIGS = {
    "C1": dict(name="DeiT-Ti 1 layer, B=4, l2 keep 50%", preset="deit_tiny", B=4, p=0.5, method="l2"),
    "C2": dict(name="DeiT-S 12 layers, B=32, p sweep", preset="deit_small", B=32, p=0.8, method="l2"),
    "C3": dict(name="DeiT-B, B=32, 80% pruned", preset="deit_base", B=32, p=0.8, method="l2"),
    "C4": dict(name="DeiT-B, B=64, 4 generators x {50,70,90}%", preset="deit_base", B=64, p=0.7, method="l2"),
    "C5": dict(name="DeiT-B, B=4096, 70% pruned, sharded", preset="deit_base", B=4096, p=0.7, method="l2"),
}
