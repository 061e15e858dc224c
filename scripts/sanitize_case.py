"""Small invocations of every kernel of libragged (both attention engines, N1, N2, N4,
the fused gather) for compute-sanitizer."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_15408_b200 as rb  # noqa: E402
import synth  # noqa: E402

for (B, N, H, p, m) in [(3, 197, 2, 0.8, "l2"), (2, 130, 1, 0.0, "all"), (4, 40, 2, 0.5, "ats")]:
    q, k, v, keep = (t.cuda() for t in synth.make_inputs(B, N, H, p, m, "bf16", seed=1))
    keep[1] = 0                                               # an empty image
    for e in (rb.ENGINE_MMA_SYNC, rb.ENGINE_TCGEN05):
        o, cu = rb.pack_attend_unpack(q, k, v, keep, want_cu=True, engine=e)
        qp, kp, vp, cu2, dst, src = rb.pack(q, k, v, keep)
        op = rb.attn(qp, kp, vp, cu2, N, engine=e)
        o2 = rb.unpack(op, dst, B, N)
# N2 mask, N1 block kernels (LN, tcgen05 GEMM x 3 epilogues, live rows), N4
# streaming attention, and the fused gather (local destinations, no signals:
# the cross-rank barrier needs concurrently running "ranks", which the
# sanitizer serialises)
import numpy as np  # noqa: E402
import oracle  # noqa: E402
x = synth.hidden_states(3, 197, 128, "bf16", seed=2).cuda()
keep2 = rb.keep_topk_l2(x, 40)
dt = torch.bfloat16
a = torch.randn(300, 256, device="cuda").to(dt)
w = (0.05 * torch.randn(384, 256, device="cuda")).to(dt)
bias = torch.zeros(384, device="cuda", dtype=dt)
res = torch.randn(300, 384, device="cuda").to(dt)
live = torch.tensor([217], dtype=torch.int32, device="cuda")
for epi in (rb.EPI_NONE, rb.EPI_GELU, rb.EPI_RESIDUAL):
    rb.linear(a, w, bias, epi, res if epi == rb.EPI_RESIDUAL else None, live=live)
y = rb.layer_norm(a, torch.ones(256, device="cuda", dtype=dt), torch.zeros(256, device="cuda", dtype=dt), live=live)
pr = synth.PRESETS["deit_tiny"]
keep3 = synth.make_inputs(3, 197, pr["H"], 0.5, "l2", "bf16", seed=3)[3].numpy()
cu3, _, _ = oracle.scan(keep3)
T3 = int(cu3[-1])
blk = rb.VitBlock({k2: v2.cuda() for k2, v2 in synth.vit_weights(pr["D"], pr["MLP"], dt, 0).items()}, 3, 197, pr["H"], dt)
xb = torch.zeros(3 * 197, pr["D"], device="cuda", dtype=dt)
xb[:T3] = synth.packed_rows(T3, pr["D"], dt, 3).cuda()
blk(xb, torch.from_numpy(cu3.astype(np.int32)).cuda())
qg = torch.randn(300 + 45, 2, 80, device="cuda").to(dt)
cug = torch.tensor([0, 300, 300, 345], dtype=torch.int32, device="cuda")
rb.attn(qg, qg, qg, cug, 300)
q, k, v, keep = (t.cuda() for t in synth.make_inputs(4, 197, 3, 0.7, "l2", "bf16", seed=4))
d0 = torch.empty(8, 197, 3, 64, device="cuda", dtype=dt)
d1 = torch.empty(8, 197, 3, 64, device="cuda", dtype=dt)
c0 = torch.empty(8, 3 * 64, device="cuda", dtype=dt)
off = 4 * 197 * 3 * 64 * 2
rb.pack_attend_unpack_gather(q, k, v, keep, rb.gather_desc(2, 1, out=[d0.data_ptr() + off, d1.data_ptr() + off],
                                                           cls=[c0.data_ptr() + 4 * 3 * 64 * 2, None]))
# round 2: the warp-specialised engine (capacity buffers from ragged_pack; N <= 256 via n_hint and
# N > 256), the block with n_hint (LayerNorm grid loop at hint 1, WS attention at hint 197), the
# EViT mask and the mask fused ahead of the scan
for (B, N, H, p) in [(3, 197, 2, 0.0), (2, 577, 2, 0.3)]:
    q, k, v, keep = (t.cuda() for t in synth.make_inputs(B, N, H, p, "random", "bf16", seed=5))
    qp, kp, vp, cu2, dst, src = rb.pack(q, k, v, keep)
    rb.attn(qp, kp, vp, cu2, N, engine=rb.ENGINE_TCGEN05_WS)
    rb.attn(qp, kp, vp, cu2, N, n_hint=N)
cud3 = torch.from_numpy(cu3.astype(np.int32)).cuda()
for hint in (1, 197):
    blk2 = rb.VitBlock({k2: v2.cuda() for k2, v2 in synth.vit_weights(pr["D"], pr["MLP"], dt, 1).items()}, 3, 197,
                       pr["H"], dt, n_hint=hint)
    blk2(xb, cud3)
q, k, v, keep = (t.cuda() for t in synth.make_inputs(3, 197, 4, 0.5, "l2", "bf16", seed=6))
rb.keep_evit(q, k, v, 60)
xh = synth.hidden_states(3, 197, 4 * 64, "bf16", seed=7).cuda()
rb.prune_l2_pack_attend_unpack(xh, q, k, v, 60)
torch.cuda.synchronize()
print("sanitize case done")
