"""Launch each kernel of the path a few times at one config for ncu.

    ncu --set full -k regex:attn_kernel -s 4 -c 2 python scripts/prof_kernels.py --config C3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2604_15408_b200 as rb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--prune", type=float, default=None)
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--engine", type=int, default=0)
ap.add_argument("--what", default="fused,attn,pack,unpack,scan")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
p = c["p"] if a.prune is None else a.prune
H = synth.PRESETS[c["preset"]]["H"]
B, N = c["B"], 197
q, k, v, keep = synth.make_inputs(B, N, H, p, c["method"], a.dtype, seed=0)
dev = torch.device("cuda")
sets = [[t.to(dev) for t in (q, k, v, keep)] for _ in range(8)]   # rotate: cold L2 per launch
outs = [torch.empty(B, N, H, 64, dtype=q.dtype, device=dev) for _ in range(8)]
cus = [torch.empty(B + 1, dtype=torch.int32, device=dev) for _ in range(8)]
what = a.what.split(",")
for i in range(a.iters):
    s = sets[i % 8]
    if "fused" in what:
        rb.pack_attend_unpack(*s, o=outs[i % 8], cu=cus[i % 8], engine=a.engine)
    if any(w in what for w in ("attn", "pack", "unpack", "scan")):
        qp, kp, vp, cu, dst, src = rb.pack(*s)
        if "attn" in what or "unpack" in what:
            op = rb.attn(qp, kp, vp, cu, N, engine=a.engine)
            rb.unpack(op, dst, B, N, o=outs[i % 8])
torch.cuda.synchronize()
print("done")
