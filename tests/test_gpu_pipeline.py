"""GPU parity of NEXT row N1's end-to-end pieces: the one-tensor
pack of the hidden state at the prune point (ragged_pack_rows, bit-exact vs
the oracle's scan + pack), the CLS readout from packed rows (ragged_cls_rows,
bit-exact), and the whole pruned forward (dense blocks -> on-device
Threshold-l2 mask -> pack -> packed blocks -> CLS) against the fp64 oracle
chained layer by layer with the same storage rounding (R22)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import bits, to_np

rb = pytest.importorskip("paper_2604_15408_b200")
pytestmark = pytest.mark.gpu
DEV = "cuda"


def _store(dtype):
    return lambda t: torch.from_numpy(np.asarray(t)).to(dtype).double().numpy()


@pytest.mark.parametrize("B,N,D,p", [(5, 197, 768, 0.7), (3, 33, 192, 0.3), (400, 197, 64, 0.5), (340, 197, 768, 0.7)])
def test_pack_rows_bitwise(B, N, D, p):
    """x [B, N, D] -> xp rows [0, T) = x[src], cu / dst / src exact (oracle.scan,
    oracle.pack); includes an empty image and a dropped CLS; B*N > 65536 takes
    the two-launch path."""
    x = synth.hidden_states(B, N, D, "bf16", seed=B)
    keep = synth.mask_random(B, N, synth.kept_tokens(N, p), seed=B)
    keep[1] = 0
    keep[2, 0] = 0
    xd = x.to(DEV)
    kd = torch.from_numpy(keep).to(DEV)
    xp, cu, dst, src = rb.pack_rows(xd, kd)
    torch.cuda.synchronize()
    rcu, rdst, rsrc = oracle.scan(keep)
    T = int(rcu[-1])
    assert cu.cpu().tolist() == rcu.tolist()
    assert dst.cpu().numpy().tolist() == rdst.tolist()
    assert src.cpu().numpy()[:T].tolist() == rsrc[:T].tolist()
    assert np.array_equal(bits(xp[:T]), bits(torch.from_numpy(oracle.pack(x.view(torch.int16).numpy(), rsrc, T)).view(torch.bfloat16)))


def test_cls_rows_bitwise():
    B, N, D = 7, 197, 384
    x = synth.hidden_states(B, N, D, "bf16", seed=3).to(DEV)
    keep = synth.mask_random(B, N, 50, seed=3)
    keep[4] = 0                                   # empty image -> +0 row
    keep[5, 0] = 0                                # dropped CLS -> its first kept row
    xp, cu, _, _ = rb.pack_rows(x, torch.from_numpy(keep).to(DEV))
    out = rb.cls_rows(xp, cu, N)
    torch.cuda.synchronize()
    c = cu.cpu().numpy()
    for b in range(B):
        want = xp[c[b]] if c[b + 1] > c[b] else torch.zeros(D, dtype=xp.dtype, device=DEV)
        assert np.array_equal(bits(out[b]), bits(want)), b


def test_pruned_forward_matches_chained_oracle():
    """DeiT-Ti shape, 6 layers pruned after layer 2 at 50 %: the GPU's CLS rows
    vs the fp64 oracle chained with bf16 storage rounding.  The oracle takes the
    GPU's keep mask (checked to be a valid Threshold-l2 top-k of the oracle's
    own prune-point state, ties within storage rounding allowed), so the
    comparison is of the same packed computation."""
    dtype = torch.bfloat16
    pr = synth.PRESETS["deit_tiny"]
    D, H, MLP, N, B, L, P = pr["D"], pr["H"], pr["MLP"], 197, 3, 6, 2
    kk = synth.kept_tokens(N, 0.5)
    layers = [synth.vit_weights(D, MLP, dtype, 100 + i) for i in range(L)]
    x0 = synth.hidden_states(B, N, D, "bf16", seed=11)
    fwd = rb.VitPrunedForward([{k: v.to(DEV) for k, v in p.items()} for p in layers], B, N, H, kk, prune_at=P)
    cls = fwd(x0.to(DEV))
    torch.cuda.synchronize()
    keep = fwd.keep.cpu().numpy()
    st = _store(dtype)
    # dense layers on all rows (cu = b*N)
    cu_all = np.arange(B + 1) * N
    x = x0.reshape(B * N, D).double().numpy()
    for i in range(P):
        x = oracle.vit_block(x, cu_all, layers[i], H, store=st)
    # the GPU mask: CLS kept, kk per image, and a valid top-k of ||x|| up to
    # the scores' storage-rounding tolerance
    assert np.all(keep.sum(1) == kk) and np.all(keep[:, 0] == 1)
    s = oracle.l2_scores(x.reshape(B, N, D))
    for b in range(B):
        kept, dropped = s[b][keep[b] == 1][1:], s[b][keep[b] == 0]
        assert kept.min() >= dropped.max() * (1 - 2.0 ** -6), b
    # packed layers
    cu, _, src = oracle.scan(keep)
    T = int(cu[-1])
    xp = x[src[:T]]
    for i in range(P, L):
        xp = oracle.vit_block(xp, cu, layers[i], H, store=st)
    ref = xp[cu[:-1]]
    got = to_np(cls)
    relf = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert relf <= 2.0 ** -7, relf
    assert np.abs(got - ref).max() <= 2.0 ** -5 * np.abs(ref).max()
