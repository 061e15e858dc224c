"""Seeded input generators: determinism, k(p) rule, mask structure, shard slices."""
import numpy as np
import torch

import synth


def test_kept_tokens_rule_values():
    """Reading R5: k(p) = N - round_half_even(p N); Table 1's 197/99/39 at
    0/50/80 % and the sweep values of SURVEY §8(c) A5."""
    want = [197, 177, 158, 138, 118, 99, 79, 59, 39, 20]
    assert [synth.kept_tokens(197, i / 10) for i in range(10)] == want
    assert synth.kept_tokens(197, 0.25) == 148


def test_activations_deterministic_and_sharded():
    a = synth.activations(6, 11, 2, 64, "bf16", seed=3)
    b = synth.activations(6, 11, 2, 64, "bf16", seed=3)
    for x, y in zip(a, b):
        assert torch.equal(x.view(torch.int16), y.view(torch.int16))
    s = synth.activations(2, 11, 2, 64, "bf16", seed=3, image_offset=4)
    for x, y in zip(a, s):
        assert torch.equal(x[4:6].view(torch.int16), y.view(torch.int16))
    v = a[2].float()
    assert v.abs().max() <= 1.0


def test_masks_structure():
    B, N = 16, 197
    for p in (0.3, 0.5, 0.8, 0.9):
        k = synth.kept_tokens(N, p)
        for fn in (synth.mask_threshold_l2, synth.mask_dynamicvit, synth.mask_random):
            m = fn(B, N, k, seed=5)
            assert m.dtype == np.uint8 and m.shape == (B, N)
            assert np.all(m[:, 0] == 1)                  # CLS always kept (R6)
            assert np.all(m.sum(1) == k)                 # uniform k
            assert np.array_equal(m, fn(B, N, k, seed=5))
        full = synth.mask_threshold_l2(B, N, k, seed=5)
        assert np.array_equal(full[3:7], synth.mask_threshold_l2(4, N, k, seed=5, image_offset=3))


def test_ats_variable_lengths_calibrated():
    B, N = 64, 197
    for p in (0.5, 0.7, 0.9):
        k = synth.kept_tokens(N, p)
        m = synth.mask_ats(B, N, k, seed=1)
        counts = m.sum(1)
        assert np.all(m[:, 0] == 1)
        assert abs(counts.mean() - k) <= 1.0
        assert counts.max() > counts.min()               # heterogeneous k_b


def test_evit_fused_token():
    q, k, v = synth.activations(4, 50, 3, 64, "bf16", seed=2)
    kk = synth.kept_tokens(50, 0.7)
    m, q2, k2, v2 = synth.mask_evit(q, k, v, kk)
    assert np.all(m.sum(1) == kk) and np.all(m[:, 0] == 1)
    for b in range(4):
        dropped = np.flatnonzero(m[b] == 0)
        j = [i for i in range(50) if i not in dropped and not torch.equal(q[b, i], q2[b, i])]
        assert len(j) == 1                               # exactly one fused row changed
        assert m[b, j[0]] == 1
        # a convex combination of dropped V rows stays inside their range
        assert v2[b, j[0]].float().abs().max() <= 1.0
