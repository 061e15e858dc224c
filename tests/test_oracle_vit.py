"""Pins of the N1 oracle (oracle/vit_block.py) against things other than
itself: torch's own LayerNorm / GELU / TransformerEncoderLayer in fp64
(library routines), GELU closed forms, and packed-image isolation."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth


def _params(D, MLP, seed=0):
    return synth.vit_weights(D, MLP, torch.bfloat16, seed)


def test_layer_norm_equals_torch_fp64():
    x = torch.randn(7, 96, dtype=torch.float64) * 3 + 1
    w, b = torch.randn(96, dtype=torch.float64), torch.randn(96, dtype=torch.float64)
    ref = torch.nn.functional.layer_norm(x, (96,), w, b, eps=oracle.LN_EPS).numpy()
    assert np.allclose(oracle.layer_norm(x, w, b), ref, rtol=0, atol=1e-12)


def test_layer_norm_invariants():
    x = np.random.default_rng(0).normal(size=(5, 64)) * 7 - 3
    y = oracle.layer_norm(x, np.ones(64), np.zeros(64))
    assert np.allclose(y.mean(axis=1), 0, atol=1e-12)
    assert np.allclose((y ** 2).mean(axis=1), 1 / (1 + oracle.LN_EPS / x.var(axis=1)), atol=1e-9)
    # shift invariance, and the affine part
    assert np.allclose(oracle.layer_norm(x + 5.0, np.ones(64), np.zeros(64)), y, atol=1e-12)
    assert np.allclose(oracle.layer_norm(x, 2 * np.ones(64), np.ones(64)), 2 * y + 1, atol=1e-12)


def test_gelu_closed_forms_and_torch():
    assert oracle.gelu(np.array([0.0]))[0] == 0.0
    assert abs(oracle.gelu(np.array([1.0]))[0] - 0.5 * (1 + math.erf(1 / math.sqrt(2)))) < 1e-15
    big = np.array([10.0, -10.0])
    assert np.allclose(oracle.gelu(big), [10.0, 0.0], atol=1e-20)
    x = torch.linspace(-6, 6, 1001, dtype=torch.float64)
    ref = torch.nn.functional.gelu(x, approximate="none").numpy()
    assert np.allclose(oracle.gelu(x), ref, rtol=0, atol=1e-15)
    # odd-part identity: gelu(x) - gelu(-x) = x
    assert np.allclose(oracle.gelu(x) - oracle.gelu(-x), x.numpy(), atol=1e-14)


def _torch_layer(params, D, H, MLP):
    layer = torch.nn.TransformerEncoderLayer(D, H, MLP, dropout=0.0, activation="gelu",
                                             layer_norm_eps=oracle.LN_EPS, batch_first=True,
                                             norm_first=True, dtype=torch.float64)
    p = {k: v.double() for k, v in params.items()}
    with torch.no_grad():
        layer.self_attn.in_proj_weight.copy_(p["w_qkv"])
        layer.self_attn.in_proj_bias.copy_(p["b_qkv"])
        layer.self_attn.out_proj.weight.copy_(p["w_proj"])
        layer.self_attn.out_proj.bias.copy_(p["b_proj"])
        layer.linear1.weight.copy_(p["w_fc1"])
        layer.linear1.bias.copy_(p["b_fc1"])
        layer.linear2.weight.copy_(p["w_fc2"])
        layer.linear2.bias.copy_(p["b_fc2"])
        layer.norm1.weight.copy_(p["ln1_w"])
        layer.norm1.bias.copy_(p["ln1_b"])
        layer.norm2.weight.copy_(p["ln2_w"])
        layer.norm2.bias.copy_(p["ln2_b"])
    layer.train()   # dropout 0; keeps torch off its fused inference fast path
    return layer


def test_block_dense_equals_torch_transformer_layer():
    """All tokens kept, one image: the oracle block == torch's pre-norm
    TransformerEncoderLayer (a library routine) in fp64."""
    D, H, MLP, n = 192, 3, 768, 37
    params = _params(D, MLP, seed=1)
    x = synth.packed_rows(n, D, seed=1)
    got = oracle.vit_block(x, np.array([0, n]), params, H)
    with torch.no_grad():
        ref = _torch_layer(params, D, H, MLP)(x.double()[None])[0].numpy()
    assert np.abs(got - ref).max() < 1e-10


def test_block_packed_equals_padded_with_key_padding_mask():
    """Pruned batch: packed rows through the oracle == torch on the padded
    batch with src_key_padding_mask, on every kept row."""
    D, H, MLP, B, N = 96, 3, 384, 3, 11
    params = _params(D, MLP, seed=2)
    rng = np.random.default_rng(2)
    keep = (rng.random((B, N)) < 0.6).astype(np.uint8)
    keep[:, 0] = 1
    xpad = synth.packed_rows(B * N, D, seed=2).reshape(B, N, D)
    cu, dst, src = oracle.scan(keep)
    T = int(cu[-1])
    xp = oracle.pack(xpad.double().numpy(), src, T)
    got = oracle.vit_block(xp, cu, params, H)
    with torch.no_grad():
        ref = _torch_layer(params, D, H, MLP)(xpad.double(),
                                               src_key_padding_mask=torch.from_numpy(keep == 0))
    ref_rows = oracle.pack(ref.numpy(), src, T)
    assert np.abs(got - ref_rows).max() < 1e-10


def test_block_isolation_and_stages():
    """Perturbing one image's rows changes no other image's output (bitwise);
    vit_block_stages ends where vit_block does."""
    D, H, MLP = 64, 1, 128
    params = _params(D, MLP, seed=3)
    cu = np.array([0, 5, 5, 12, 13])            # includes an empty image
    x = synth.packed_rows(13, D, seed=3).double().numpy()
    base = oracle.vit_block(x, cu, params, H)
    x2 = x.copy()
    x2[5:12] += 1.0
    pert = oracle.vit_block(x2, cu, params, H)
    assert (pert[:5] == base[:5]).all() and (pert[12:] == base[12:]).all()
    assert not np.allclose(pert[5:12], base[5:12])
    st = oracle.vit_block_stages(x, cu, params, H)
    assert (st["out"] == base).all()
    assert st["qkv"].shape == (13, 3 * D) and st["f"].shape == (13, MLP)


def test_block_store_rounding_points():
    """With a bf16 store the result differs from pure fp64 by rounding-sized
    amounts only (the store hook is applied, and nowhere catastrophically)."""
    D, H, MLP = 128, 2, 512
    params = _params(D, MLP, seed=4)
    cu = np.array([0, 20, 31])
    x = synth.packed_rows(31, D, seed=4)
    bf = lambda t: torch.from_numpy(np.asarray(t)).to(torch.bfloat16).double().numpy()  # noqa: E731
    a = oracle.vit_block(x, cu, params, H)
    b = oracle.vit_block(x, cu, params, H, store=bf)
    err = np.abs(a - b).max()
    assert 0 < err < 0.1 * np.abs(a).max()
    assert (bf(b) == b).all()                    # the output itself is stored
