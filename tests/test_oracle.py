"""Pins for the fp64 oracle (-m "not gpu").  Each test checks the oracle against
something other than itself: a value the paper (or SPEC) prints, a closed form,
a library routine, brute force, or an invariant fixed by the mathematics."""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from conftest import GOLDEN


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- scan ----

def test_scan_spec_worked_example():
    g = _golden("spec_scan_examples.json")["cases"][0]
    cu, dst, src = oracle.scan(np.array(g["keep"], np.uint8))
    assert cu.tolist() == g["cu"]
    assert dst.tolist() == g["dst"]
    assert src[: cu[-1]].tolist() == g["src"]


def test_scan_all_true_spec():
    g = _golden("spec_scan_examples.json")["cases"][1]
    B, N = g["all_true"]["B"], g["all_true"]["N"]
    cu, dst, src = oracle.scan(np.ones((B, N), np.uint8))
    assert cu.tolist() == g["cu"]
    assert src.tolist() == list(range(B * N))
    assert dst.tolist() == list(range(B * N))


def test_table1_token_counts_and_totals():
    """Table 1 Tok/img and the T totals of P:202 / P:238."""
    g = _golden("paper_table1.json")
    for row in g["tokens_per_image"]:
        k = synth.kept_tokens(197, row["prune"])
        assert k == row["tok"], row
        keep = synth.mask_threshold_l2(row["bs"], 197, k, seed=7)
        cu, _, _ = oracle.scan(keep)
        assert np.all(np.diff(cu) == row["tok"])
    for row in g["total_tokens"]:
        keep = synth.mask_threshold_l2(row["bs"], 197, synth.kept_tokens(197, row["prune"]), 1)
        assert oracle.scan(keep)[0][-1] == row["T"]
    # 80 % pruning leaves (39/197)^2 ~ 0.04 of the attention FLOPs
    assert abs((39 / 197) ** 2 - g["flop_ratio_80pct"]["value"]) < 2e-3


def test_scan_brute_force_global_rank():
    """dst of a kept token = number of kept tokens before it in flattened
    (image-major, position-minor) order; every mask over B=2, N<=6."""
    for N in range(1, 7):
        for bits in itertools.product([0, 1], repeat=2 * N):
            keep = np.array(bits, np.uint8).reshape(2, N)
            cu, dst, src = oracle.scan(keep)
            flat = keep.reshape(-1)
            for i in range(2 * N):
                want = sum(int(flat[j]) for j in range(i)) if flat[i] else -1
                assert dst[i] == want
            for b in range(2):
                assert cu[b + 1] - cu[b] == sum(int(x) for x in keep[b])
            T = int(cu[-1])
            assert sorted(src[:T].tolist()) == src[:T].tolist()
            assert all(dst[src[r]] == r for r in range(T))


def test_scan_matches_library_routines():
    """torch.nonzero (indices) and flash_attn.bert_padding.unpad_input
    (cu_seqlens, indices, max_seqlen) on random masks with empty images."""
    bert_padding = pytest.importorskip("flash_attn.bert_padding")
    rng = np.random.default_rng(3)
    for trial in range(20):
        B, N = int(rng.integers(1, 9)), int(rng.integers(1, 40))
        keep = (rng.random((B, N)) < rng.random()).astype(np.uint8)
        cu, dst, src = oracle.scan(keep)
        T = int(cu[-1])
        nz = torch.nonzero(torch.from_numpy(keep).reshape(-1)).reshape(-1)
        assert src[:T].tolist() == nz.tolist()
        x = torch.arange(B * N, dtype=torch.float32).reshape(B, N, 1)
        out = bert_padding.unpad_input(x, torch.from_numpy(keep).bool())
        x_unpad, indices, cu_lib, max_len = out[0], out[1], out[2], out[3]
        assert cu_lib.tolist() == cu.tolist()
        assert indices.tolist() == src[:T].tolist()
        assert max_len == (int(np.diff(cu).max()) if B else 0)


def test_validate_cu_seqlens_examples():
    g = _golden("spec_scan_examples.json")

    def valid(cu, T):
        return cu[0] == 0 and all(a <= b for a, b in zip(cu, cu[1:])) and cu[-1] == T
    for c in g["valid_cu"]:
        assert valid(c["cu"], c["T"])
    for c in g["invalid_cu"]:
        assert not valid(c["cu"], c["T"])
    rng = np.random.default_rng(0)
    for _ in range(10):
        keep = (rng.random((5, 17)) < 0.4).astype(np.uint8)
        cu = oracle.scan(keep)[0]
        assert valid(cu.tolist(), int(keep.sum()))


# ------------------------------------------------------- pack / unpack ----

def _bits(t):
    return t.contiguous().view(torch.int16).numpy()


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_pack_unpack_roundtrip_bitwise(dtype):
    q, _, _, keep = synth.make_inputs(3, 33, 2, 0.6, "random", dtype, seed=4)
    cu, dst, src = oracle.scan(keep.numpy())
    T = int(cu[-1])
    qb = _bits(q)
    packed = oracle.pack(qb, src, T)
    back = oracle.unpack(packed, dst, 3, 33, 0)
    km = keep.numpy().astype(bool)
    assert np.array_equal(back[km], qb[km])                 # kept rows: identity
    assert np.all(back[~km] == 0)                           # dropped rows: +0.0 bits
    for b in range(3):                                      # CLS at packed row cu[b]
        assert np.array_equal(packed[cu[b]], qb[b, 0])
    # order preservation: packed rows of image b appear in ascending position
    for b in range(3):
        assert np.all(np.diff(src[cu[b]:cu[b + 1]]) > 0)


def test_pack_all_true_is_identity():
    q, _, _ = synth.activations(2, 9, 3, 64, "bf16", 1)
    cu, dst, src = oracle.scan(np.ones((2, 9), np.uint8))
    qb = _bits(q)
    assert np.array_equal(oracle.pack(qb, src, 18), qb.reshape(18, 3, 64))
    assert np.array_equal(oracle.unpack(oracle.pack(qb, src, 18), dst, 2, 9), qb)


def test_unpack_matches_flash_attn_pad_input():
    bert_padding = pytest.importorskip("flash_attn.bert_padding")
    rng = np.random.default_rng(5)
    keep = (rng.random((4, 21)) < 0.5).astype(np.uint8)
    keep[:, 0] = 1
    cu, dst, src = oracle.scan(keep)
    T = int(cu[-1])
    op = rng.standard_normal((T, 2, 8))
    ours = oracle.unpack(op, dst, 4, 21, 0.0)
    ref = bert_padding.pad_input(torch.from_numpy(op.reshape(T, 16)),
                                 torch.from_numpy(src[:T]), 4, 21)
    assert np.array_equal(ours.reshape(4, 21, 16), ref.numpy())


# ---------------------------------------------------------- attention ----

def test_attention_single_token_returns_v():
    """n = 1: softmax over one key is 1, output = that V row."""
    rng = np.random.default_rng(0)
    q, k, v = rng.standard_normal((3, 1, 64))
    assert np.array_equal(oracle.attention_one(q, k, v), v)


def test_attention_identical_keys_gives_column_mean():
    """All keys identical -> uniform weights -> column mean of V."""
    rng = np.random.default_rng(1)
    n = 13
    q = rng.standard_normal((n, 64))
    k = np.repeat(rng.standard_normal((1, 64)), n, axis=0)
    v = rng.standard_normal((n, 64))
    np.testing.assert_allclose(oracle.attention_one(q, k, v),
                               np.repeat(v.mean(0, keepdims=True), n, 0), rtol=0, atol=1e-13)


def test_attention_two_token_closed_form():
    """n = 2: o_i = sigma(s_i1 - s_i2) v_1 + sigma(s_i2 - s_i1) v_2."""
    rng = np.random.default_rng(2)
    q, k, v = rng.standard_normal((3, 2, 64))
    s = np.array([[q[i] @ k[j] / 8.0 for j in range(2)] for i in range(2)])
    sig = lambda x: 1.0 / (1.0 + math.exp(-x))  # noqa: E731
    want = np.stack([sig(s[i, 0] - s[i, 1]) * v[0] + sig(s[i, 1] - s[i, 0]) * v[1] for i in range(2)])
    np.testing.assert_allclose(oracle.attention_one(q, k, v), want, rtol=0, atol=1e-14)


def test_attention_dense_equals_torch_sdpa_fp64():
    """0 % pruning == dense SDPA (library routine, fp64 CPU) per image and head."""
    q, k, v, keep = synth.make_inputs(2, 197, 3, 0.0, "all", "bf16", seed=9)
    o, cu = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.double().transpose(1, 2), k.double().transpose(1, 2), v.double().transpose(1, 2)
    ).transpose(1, 2).numpy()
    np.testing.assert_allclose(o, ref, rtol=0, atol=1e-12)
    assert cu.tolist() == [0, 197, 394]


def test_attention_pruned_equals_masked_sdpa_fp64():
    """Ragged == padded SDPA with a key-padding mask on kept query rows."""
    q, k, v, keep = synth.make_inputs(3, 40, 2, 0.7, "random", "fp16", seed=10, dist="peaked")
    o, _ = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    mask = keep.bool()[:, None, None, :]
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.double().transpose(1, 2), k.double().transpose(1, 2), v.double().transpose(1, 2),
        attn_mask=mask).transpose(1, 2).numpy()
    km = keep.numpy().astype(bool)
    np.testing.assert_allclose(o[km], ref[km], rtol=0, atol=1e-12)
    assert np.all(o[~km] == 0.0)


def test_attention_matches_scipy_logsumexp():
    scipy_special = pytest.importorskip("scipy.special")
    rng = np.random.default_rng(11)
    q, k, v = rng.standard_normal((3, 23, 64)) * np.array([3.0, 3.0, 1.0])[:, None, None]
    S = q @ k.T / 8.0
    lse = scipy_special.logsumexp(S, axis=1, keepdims=True)
    np.testing.assert_allclose(oracle.attention_one(q, k, v), np.exp(S - lse) @ v, rtol=0, atol=1e-12)


def test_softmax_rows_sum_to_one():
    rng = np.random.default_rng(12)
    P = oracle.softmax_weights(rng.standard_normal((31, 64)) * 3, rng.standard_normal((31, 64)))
    np.testing.assert_allclose(P.sum(1), 1.0, rtol=0, atol=1e-14)
    assert np.all(P >= 0)


def test_permutation_equivariance():
    rng = np.random.default_rng(13)
    q, k, v = rng.standard_normal((3, 17, 64))
    perm = rng.permutation(17)
    a = oracle.attention_one(q, k, v)[perm]
    b = oracle.attention_one(q[perm], k[perm], v[perm])
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-13)


def test_cross_image_isolation_bitwise():
    q, k, v, keep = synth.make_inputs(3, 30, 2, 0.5, "random", "bf16", seed=14)
    o1, _ = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    q2, k2, v2 = q.clone(), k.clone(), v.clone()
    q2[1] = -q2[1]
    v2[1] = v2[1] * 0.5
    o2, _ = oracle.pack_attend_unpack(q2, k2, v2, keep.numpy())
    assert np.array_equal(o1[0], o2[0]) and np.array_equal(o1[2], o2[2])
    assert not np.array_equal(o1[1], o2[1])


def _alg1_tiled(q, k, v, BM, BN):
    """Alg. 1 transcribed for one (image, head): q-tile loop, kv-tile
    loop, online softmax with running (m, l, o), final o / l.  Tail tiles mask
    key columns >= n to -inf and drop query rows >= n (reading R4)."""
    n, d = q.shape
    out = np.zeros((n, d))
    for m0 in range(0, n, BM):
        qt = q[m0:m0 + BM]
        m = np.full(qt.shape[0], -np.inf)
        l = np.zeros(qt.shape[0])
        o = np.zeros((qt.shape[0], d))
        for j0 in range(0, n, BN):
            kt, vt = k[j0:j0 + BN], v[j0:j0 + BN]
            S = qt @ kt.T / math.sqrt(d)
            m_new = np.maximum(m, S.max(1))
            alpha = np.exp(m - m_new)
            P = np.exp(S - m_new[:, None])
            o = alpha[:, None] * o + P @ vt
            l = alpha * l + P.sum(1)
            m = m_new
        out[m0:m0 + BM] = o / l[:, None]
    return out


@pytest.mark.parametrize("n", [1, 5, 39, 64, 65, 100, 197])
@pytest.mark.parametrize("tile", [8, 16, 64])
def test_alg1_online_softmax_equals_plain(n, tile):
    """Alg. 1 is an exact reformulation of the plain softmax the oracle computes
    (FA2 online softmax): tile-size invariance."""
    rng = np.random.default_rng(n * 100 + tile)
    q, k, v = rng.standard_normal((3, n, 64)) * np.array([3.0, 3.0, 1.0])[:, None, None]
    np.testing.assert_allclose(_alg1_tiled(q, k, v, tile, tile), oracle.attention_one(q, k, v),
                               rtol=0, atol=1e-12)


def test_empty_image_and_composition():
    """n = 0 images produce no packed rows and all-zero padded rows (R11);
    the fused oracle equals unpack o attention o pack."""
    q, k, v, keep = synth.make_inputs(4, 25, 2, 0.5, "random", "bf16", seed=15)
    keep = keep.numpy().copy()
    keep[2] = 0
    o, cu = oracle.pack_attend_unpack(q, k, v, keep)
    assert cu[3] == cu[2]
    assert np.all(o[2] == 0.0)
    c, dst, src = oracle.scan(keep)
    T = int(c[-1])
    f64 = [oracle.as_f64(t) for t in (q, k, v)]
    op = oracle.attention(*(oracle.pack(t, src, T) for t in f64), c)
    assert np.array_equal(o, oracle.unpack(op, dst, 4, 25, 0.0))


def test_oracle_rejects_nonfinite():
    x = np.zeros((3, 1, 64))
    x[1, 0, 0] = np.nan
    with pytest.raises(ValueError):
        oracle.attention(x, x, x, np.array([0, 3]))


# ------------------------------------------------- N2: Threshold-l2 mask ----

def test_keep_topk_l2_brute_force():
    """Brute force on tiny inputs: the kept set is CLS plus the k-1 positions
    with the largest ||x||, ties to the lower index (checked by enumerating
    every subset of size k-1 and picking the lexicographic best)."""
    rng = np.random.default_rng(21)
    for trial in range(30):
        N, D = int(rng.integers(2, 8)), int(rng.integers(1, 5))
        x = np.round(rng.standard_normal((1, N, D)) * 2) / 2        # exact ties happen
        k = int(rng.integers(1, N + 1))
        got = oracle.keep_topk_l2(x, k)[0]
        norms = [math.sqrt(sum(v * v for v in x[0, n])) for n in range(N)]
        best = None
        for subset in itertools.combinations(range(1, N), k - 1):
            key = (sorted((-norms[n], n) for n in subset))
            if best is None or key < best[0]:
                best = (key, subset)
        want = np.zeros(N, np.uint8)
        want[0] = 1
        want[list(best[1])] = 1
        assert np.array_equal(got, want), (x, k)


def test_keep_topk_l2_invariants_and_table1_counts():
    x = synth.hidden_states(8, 197, 64, "bf16", seed=3)
    for p, tok in ((0.0, 197), (0.5, 99), (0.8, 39)):                 # Table 1
        keep = oracle.keep_topk_l2(x, synth.kept_tokens(197, p))
        assert np.all(keep.sum(1) == tok) and np.all(keep[:, 0] == 1)
        s = oracle.l2_scores(x)
        for b in range(8):
            kept, dropped = s[b][keep[b] == 1], s[b][keep[b] == 0]
            if dropped.size:
                assert kept.min() >= dropped.max()                      # threshold property


# ---------------------------------------------- N4: FP8 E4M3 decode (R23) ----

def test_e4m3_decode_matches_torch_for_every_byte():
    """The oracle's formula decode vs torch.float8_e4m3fn (library routine),
    all 256 bytes (NaN at 0x7f / 0xff)."""
    b = np.arange(256, dtype=np.uint8)
    ref = torch.from_numpy(b).view(torch.float8_e4m3fn).double().numpy()
    got = oracle.e4m3_decode(b)
    assert np.array_equal(np.isnan(got), np.isnan(ref)) and np.isnan(got).sum() == 2
    ok = ~np.isnan(ref)
    assert np.array_equal(got[ok], ref[ok])


def test_e4m3_decode_closed_forms():
    d = oracle.e4m3_decode(np.array([0x00, 0x80, 0x38, 0xB8, 0x7E, 0x01, 0x08, 0x07, 0x40], np.uint8))
    assert d.tolist() == [0.0, -0.0, 1.0, -1.0, 448.0, 2.0 ** -9, 2.0 ** -6, 7 * 2.0 ** -9, 2.0]


def test_attention_fp8_is_attention_of_dequantised_inputs():
    """attention_fp8 == attention on the decoded, scaled values; scaling V by
    c scales O by c exactly (the oracle's fp64 arithmetic on dyadic scales)."""
    rng = np.random.default_rng(3)
    q8, k8, v8 = (rng.integers(0, 0x7E, size=(7, 2, 32), dtype=np.uint8) for _ in range(3))
    cu = np.array([0, 3, 7])
    a = oracle.attention_fp8(q8, k8, v8, (0.5, 0.25, 2.0), cu)
    b = oracle.attention(oracle.e4m3_decode(q8) * 0.5, oracle.e4m3_decode(k8) * 0.25,
                         oracle.e4m3_decode(v8) * 2.0, cu)
    assert np.array_equal(a, b)
    c = oracle.attention_fp8(q8, k8, v8, (0.5, 0.25, 4.0), cu)
    assert np.array_equal(c, 2.0 * a)


# ------------------------------------ round-2 pins for the helper functions ----

def _sdpa64(q, k, v, mask=None):
    """torch SDPA in fp64 on [n, d] (library routine; default scale 1/sqrt(d))."""
    t = [torch.as_tensor(np.asarray(x, np.float64))[None, None] for x in (q, k, v)]
    return torch.nn.functional.scaled_dot_product_attention(*t, attn_mask=mask)[0, 0].numpy()


def test_attention_image_head_equals_masked_sdpa_for_every_image_and_head():
    """attention_image_head(b, h) -- the C5 sampled checker -- against torch
    SDPA in fp64 on the padded (b, h) slice with a key-padding mask (P:40-42:
    padded attention with masks computes the same kept rows), for every (b, h)
    of a ragged batch that includes an empty image and a CLS-only image; and
    against the whole-path oracle on the same rows."""
    B, N, H = 5, 23, 3
    q, k, v, keep = synth.make_inputs(B, N, H, 0.6, "random", "bf16", seed=21, dist="peaked")
    keep = keep.numpy().copy()
    keep[1] = 0                       # empty image
    keep[3] = 0
    keep[3, 0] = 1                    # CLS only
    o, _ = oracle.pack_attend_unpack(q, k, v, keep)
    for b in range(B):
        kb = keep[b].astype(bool)
        for h in range(H):
            pos, rows = oracle.attention_image_head(q, k, v, keep, b, h)
            assert pos.tolist() == np.flatnonzero(kb).tolist()
            assert rows.shape == (kb.sum(), 64)
            if kb.sum() == 0:
                continue
            mask = torch.as_tensor(kb)[None, None, None, :]
            ref = _sdpa64(q[b, :, h].double(), k[b, :, h].double(), v[b, :, h].double(), mask)[kb]
            np.testing.assert_allclose(rows, ref, rtol=0, atol=1e-12)
            np.testing.assert_array_equal(rows, o[b, pos, h])
    # a wrong head or image selection must not pass: neighbouring heads differ
    _, r0 = oracle.attention_image_head(q, k, v, keep, 0, 0)
    _, r1 = oracle.attention_image_head(q, k, v, keep, 0, 1)
    assert np.abs(r0 - r1).max() > 1e-3


@pytest.mark.parametrize("d", [64, 32, 80])
def test_softmax_weights_equals_torch_softmax_and_reproduces_attention(d):
    """softmax_weights(q, k) == torch.softmax(q k^T / sqrt(d)) in fp64 (library
    routine; a wrong 1/sqrt(d) fails, which rows-sum-to-one alone would not
    catch), and softmax_weights(q, k) @ v == SDPA(q, k, v)."""
    rng = np.random.default_rng(22 + d)
    q, k, v = rng.standard_normal((3, 29, d)) * np.array([3.0, 1.0, 1.0])[:, None, None]
    P = oracle.softmax_weights(q, k)
    ref = torch.softmax(torch.as_tensor(q) @ torch.as_tensor(k).T / math.sqrt(d), dim=1).numpy()
    np.testing.assert_allclose(P, ref, rtol=0, atol=1e-14)
    np.testing.assert_allclose(P @ v, _sdpa64(q, k, v), rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.attention_one(q, k, v), _sdpa64(q, k, v), rtol=0, atol=1e-12)


def test_attention_fp8_equals_torch_float8_dequant_sdpa():
    """attention_fp8 by an independent route: the bytes viewed as
    torch.float8_e4m3fn (library decode), widened to fp64, multiplied by the
    descales in torch, then torch SDPA in fp64 per image (P:286-326 applied to
    the dequantised values, R23).  Includes subnormal and max-magnitude bytes."""
    rng = np.random.default_rng(23)
    T, H, d = 13, 2, 32
    q8, k8, v8 = (rng.integers(0, 256, size=(T, H, d), dtype=np.uint8) for _ in range(3))
    for t in (q8, k8, v8):          # no NaN bytes (0x7f / 0xff): parity is on finite inputs
        t[(t & 0x7F) == 0x7F] = 0x7E
    q8[0, 0, :4] = [0x01, 0x81, 0x07, 0x7E]         # subnormals and 448
    cu = np.array([0, 1, 1, 6, 13])                   # n = 1, an empty image, 5, 7
    desc = (0.03125, 0.0625, 1.5)
    got = oracle.attention_fp8(q8, k8, v8, desc, cu)

    def deq(b, s):
        return torch.from_numpy(b).view(torch.float8_e4m3fn).to(torch.float64) * s

    tq, tk, tv = deq(q8, desc[0]), deq(k8, desc[1]), deq(v8, desc[2])
    for i in range(len(cu) - 1):
        s, e = int(cu[i]), int(cu[i + 1])
        for h in range(H):
            if e == s:
                continue
            ref = torch.nn.functional.scaled_dot_product_attention(
                tq[s:e, h][None, None], tk[s:e, h][None, None], tv[s:e, h][None, None])[0, 0].numpy()
            np.testing.assert_allclose(got[s:e, h], ref, rtol=0, atol=1e-9 * max(1.0, np.abs(ref).max()))


def test_keep_topk_l2_rejects_k_below_one_and_ranks_nan_last():
    """CLS always survives (R6): k < 1 is an error; a NaN score ranks below every
    finite one, so at most k tokens are kept (R20)."""
    x = np.ones((1, 5, 4))
    x[0, 2] = np.nan
    with pytest.raises(ValueError):
        oracle.keep_topk_l2(x, 0)
    assert oracle.keep_topk_l2(x, 4)[0].tolist() == [1, 1, 0, 1, 1]
    assert oracle.keep_topk_l2(x, 5)[0].tolist() == [1, 1, 1, 1, 1]


# ------------------------------------------- N2: EViT keep mask (R17) ----

def _evit_logits_loops(q, k):
    """Independent triple loop in plain Python floats (not the oracle's matmuls)."""
    B, N, H, d = k.shape
    out = [[0.0] * N for _ in range(B)]
    for b in range(B):
        for n in range(N):
            acc = 0.0
            for h in range(H):
                acc += sum(float(q[b, 0, h, c]) * float(k[b, n, h, c]) for c in range(d)) / math.sqrt(d)
            out[b][n] = acc / H
    return np.array(out)


def test_evit_logits_equal_loops_and_cls_attention_of_sdpa():
    """evit_logits against (i) plain loops and (ii) the CLS row of torch's fp64
    attention logits q k^T / sqrt(d) (SDPA's own scale), head-averaged."""
    q, k, v, _ = synth.make_inputs(2, 9, 3, 0.0, "all", "bf16", seed=31, d=16)
    got = oracle.evit_logits(q, k)
    np.testing.assert_allclose(got, _evit_logits_loops(q.double().numpy(), k.double().numpy()), rtol=0, atol=1e-12)
    qt, kt = q.double().transpose(1, 2), k.double().transpose(1, 2)          # [B, H, N, d]
    S = (qt @ kt.transpose(-1, -2)) / math.sqrt(16)                            # SDPA's logits
    np.testing.assert_allclose(got, S[:, :, 0, :].mean(1).numpy(), rtol=0, atol=1e-12)


def test_keep_evit_brute_force():
    """Tiny inputs, every k: the kept non-CLS, non-fused set is the lexicographic
    best (logit desc, index asc) subset of size k-2 over all subsets of 1..N-1
    (brute force on loop logits); the fused token sits in the first dropped
    position and equals the softmax(logit)-weighted mean of ALL dropped rows,
    computed here row by row."""
    rng = np.random.default_rng(32)
    for trial in range(25):
        N, H, d = int(rng.integers(3, 8)), int(rng.integers(1, 3)), 4
        q = np.round(rng.standard_normal((1, N, H, d)) * 2) / 2       # ties happen
        k = np.round(rng.standard_normal((1, N, H, d)) * 2) / 2
        v = rng.standard_normal((1, N, H, d))
        kk = int(rng.integers(1, N + 1))
        keep, f, fused = oracle.keep_evit(q, k, v, kk)
        lg = _evit_logits_loops(q, k)[0]
        if kk >= N:
            assert keep[0].tolist() == [1] * N and f[0] == -1
            continue
        best = None
        for subset in itertools.combinations(range(1, N), max(kk - 2, 0)):
            key = sorted((-lg[n], n) for n in subset)
            if best is None or key < best[0]:
                best = (key, subset)
        chosen = {0, *best[1]}
        dropped = [n for n in range(N) if n not in chosen]
        want = np.zeros(N, np.uint8)
        want[list(chosen)] = 1
        if kk >= 2:
            want[dropped[0]] = 1
            assert f[0] == dropped[0]
            w = [math.exp(lg[j] - max(lg[i] for i in dropped)) for j in dropped]
            z = sum(w)
            for t, x in enumerate((q, k, v)):
                ref = sum(wj / z * x[0, j] for wj, j in zip(w, dropped))
                np.testing.assert_allclose(fused[0, t], ref, rtol=0, atol=1e-12)
        else:
            assert f[0] == -1
        assert keep[0].tolist() == want.tolist(), (kk, lg)
        assert keep[0].sum() == min(kk, N)


def test_keep_evit_closed_forms_and_generator_agreement():
    """Equal logits -> the lowest positions kept and the fused token is the plain
    mean of the dropped rows; identical dropped rows -> the fused token equals
    that row exactly (weights sum to 1); and agreement with the independent
    host generator synth.mask_evit (same reading R17, separate code)."""
    B, N, H, d = 1, 10, 2, 8
    q = np.zeros((B, N, H, d))                       # CLS query 0 -> every logit 0
    rng = np.random.default_rng(33)
    k, v = rng.standard_normal((2, B, N, H, d))
    keep, f, fused = oracle.keep_evit(q, k, v, 5)
    assert keep[0].tolist() == [1, 1, 1, 1, 1, 0, 0, 0, 0, 0] and f[0] == 4
    np.testing.assert_allclose(fused[0, 2], v[0, 4:].mean(0), rtol=0, atol=1e-14)
    q2, k2 = rng.standard_normal((2, B, N, H, d))
    v2 = v.copy()
    v2[0, 1:] = v2[0, 9]                              # every non-CLS row identical
    keep2, f2, fused2 = oracle.keep_evit(q2, k2, v2, 4)
    assert f2[0] > 0 and keep2[0].sum() == 4
    assert np.abs(fused2[0, 2] - v2[0, 9]).max() < 1e-14
    # the host generator (bf16 inputs, fused rows rounded to bf16)
    q, k, v, _ = synth.make_inputs(3, 40, 3, 0.0, "all", "bf16", seed=34)
    for kk in (2, 9, 21, 39):
        mask, qs, ks, vs = synth.mask_evit(q, k, v, kk)
        keep, f, fused = oracle.keep_evit(q, k, v, kk)
        assert np.array_equal(mask, keep), kk
        for b in range(3):
            if f[b] >= 0:
                for t, x in enumerate((qs, ks, vs)):
                    ref = torch.from_numpy(fused[b, t]).to(torch.bfloat16).double().numpy()
                    np.testing.assert_array_equal(x[b, f[b]].double().numpy(), ref)
