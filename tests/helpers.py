"""Shared test helpers: tolerances (R2) and oracle comparisons."""
import numpy as np
import torch

import oracle

# BASELINE.json north_star: max-abs vs the fp64 oracle
TOL = {torch.bfloat16: 2e-3, torch.float16: 5e-4}
MANT = {torch.bfloat16: 7, torch.float16: 10}


def ulp(x: np.ndarray, dtype) -> np.ndarray:
    """ulp of |x| in the 16-bit output type (normal range; fp16 subnormal floor)."""
    ax = np.maximum(np.abs(x), 2.0 ** -24)
    e = np.floor(np.log2(ax))
    u = 2.0 ** (e - MANT[dtype])
    return np.maximum(u, 2.0 ** -24 if dtype == torch.float16 else 0.0)


def check_attention(got_f64: np.ndarray, ref: np.ndarray, dtype, vmax=None, dist="standard"):
    """Primary bound (standard/peaked, |V| < 1): max-abs <= 2e-3 / 5e-4.
    Secondary bound (any distribution): |err| <= ulp(|ref|) + 2^-12 max|V|."""
    err = np.abs(got_f64 - ref)
    if dist in ("standard", "peaked"):
        assert err.max(initial=0.0) <= TOL[dtype], f"max-abs {err.max():.3e} > {TOL[dtype]}"
    vm = 1.0 if vmax is None else vmax
    bound = ulp(ref, dtype) + 2.0 ** -12 * vm
    ratio = (err / bound).max(initial=0.0)
    assert ratio <= 1.0, f"secondary bound exceeded: worst ratio {ratio:.3f}"
    return float(err.max(initial=0.0))


def bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().view(torch.int16).cpu().numpy()


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().double().numpy()


def fused_oracle(q, k, v, keep):
    """fp64 oracle of the whole path on CPU copies."""
    return oracle.pack_attend_unpack(q.cpu(), k.cpu(), v.cpu(), keep.cpu().numpy())
