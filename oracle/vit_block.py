"""fp64 CPU oracle of NEXT row N1: one pre-norm ViT block on PACKED rows.

TEST INFRASTRUCTURE ONLY (same rule as ragged_oracle.py: only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import it; it imports nothing from the product package).

Passages followed:
  P:355-370 "End-to-End Pipeline Integration": after the pruning point the
            packed buffer + cu_seqlens feed "ragged attention + MLP on packed
            buffer" for layers 5-12, and the CLS token is read from the packed
            buffer (row cu[b] of image b).
  P:449-451: the MLP is where end-to-end time goes once attention
            is ragged.
  The block itself is the DeiT/timm pre-norm block the paper runs (P:137
  timm 1.0): x + proj(attn(LN1(x))), then + fc2(GELU(fc1(LN2(x)))), with
  LayerNorm eps 1e-6 and exact (erf) GELU -- DESIGN.md reading R21.
  Attention is ragged_oracle.attention (Alg. 1's plain form) over cu_seqlens.

Storage precision (R22): the GPU path stores every intermediate
activation in the 16-bit input dtype between kernels (LN outputs, qkv,
attention output, the residual stream, the GELU output).  `vit_block(...,
store=...)` applies a rounding function at exactly those points (identity =
pure fp64); everything between them is fp64.  The rounding function is the
caller's (numpy/torch dtype casts), not method arithmetic.

Pins (tests/test_oracle.py): torch.nn.functional.layer_norm and gelu in fp64,
GELU closed-form values, the whole block against torch's
nn.TransformerEncoderLayer (norm_first, gelu, eps 1e-6) in fp64 on one dense
image and on a padded batch with src_key_padding_mask (kept rows), and
packed-image isolation.
"""
from __future__ import annotations

import math

import numpy as np

from .ragged_oracle import as_f64, attention

LN_EPS = 1e-6  # DeiT / timm LayerNorm eps (R21)


def layer_norm(x, w, b, eps: float = LN_EPS) -> np.ndarray:
    """Row-wise LayerNorm: (x - mean) / sqrt(var + eps) * w + b, biased variance."""
    x = as_f64(x)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * as_f64(w) + as_f64(b)


_erf = np.vectorize(math.erf, otypes=[np.float64])


def gelu(x) -> np.ndarray:
    """Exact GELU: x * Phi(x) = 0.5 x (1 + erf(x / sqrt 2))."""
    x = as_f64(x)
    return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))


def linear(x, w, b) -> np.ndarray:
    """y = x W^T + b, W [out, in] (the torch / timm layout)."""
    return as_f64(x) @ as_f64(w).T + as_f64(b)


def vit_block(x, cu, params: dict, H: int, store=None) -> np.ndarray:
    """One block on packed rows x [T, D] with per-image row ranges cu [B+1].

    y = LN1(x); qkv = y Wqkv^T + bqkv viewed [T, 3, H, d] (q|k|v, head, d);
    a = attention(q, k, v, cu) per image and head; h = x + a Wproj^T + bproj;
    z = LN2(h); f = GELU(z Wfc1^T + bfc1); out = h + f Wfc2^T + bfc2.
    `store` rounds at the storage points (R22); None = fp64 throughout."""
    r = (lambda t: t) if store is None else store
    x = as_f64(x)
    T, D = x.shape
    d = D // H
    p = {k: as_f64(v) for k, v in params.items()}
    y = r(layer_norm(x, p["ln1_w"], p["ln1_b"]))
    qkv = r(linear(y, p["w_qkv"], p["b_qkv"])).reshape(T, 3, H, d)
    a = r(attention(qkv[:, 0], qkv[:, 1], qkv[:, 2], np.asarray(cu)).reshape(T, D))
    h = r(x + linear(a, p["w_proj"], p["b_proj"]))
    z = r(layer_norm(h, p["ln2_w"], p["ln2_b"]))
    f = r(gelu(linear(z, p["w_fc1"], p["b_fc1"])))
    return r(h + linear(f, p["w_fc2"], p["b_fc2"]))


def vit_block_stages(x, cu, params: dict, H: int, store=None) -> dict:
    """Same computation as vit_block, returning every stored intermediate
    (for per-kernel parity tests): y, qkv [T, 3D], a, h, z, f, out."""
    r = (lambda t: t) if store is None else store
    x = as_f64(x)
    T, D = x.shape
    d = D // H
    p = {k: as_f64(v) for k, v in params.items()}
    s = {}
    s["y"] = r(layer_norm(x, p["ln1_w"], p["ln1_b"]))
    s["qkv"] = r(linear(s["y"], p["w_qkv"], p["b_qkv"]))
    q3 = s["qkv"].reshape(T, 3, H, d)
    s["a"] = r(attention(q3[:, 0], q3[:, 1], q3[:, 2], np.asarray(cu)).reshape(T, D))
    s["h"] = r(x + linear(s["a"], p["w_proj"], p["b_proj"]))
    s["z"] = r(layer_norm(s["h"], p["ln2_w"], p["ln2_b"]))
    s["f"] = r(gelu(linear(s["z"], p["w_fc1"], p["b_fc1"])))
    s["out"] = r(s["h"] + linear(s["f"], p["w_fc2"], p["b_fc2"]))
    return s
