"""Small invocations of every kernel (both engines) for compute-sanitizer."""
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
torch.cuda.synchronize()
print("sanitize case done")
