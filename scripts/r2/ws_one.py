"""One configuration of ragged_attn for ncu captures: --case vitl|c3p0|n1024 --engine 3"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_15408_b200 as rb
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--case", default="vitl")
ap.add_argument("--engine", type=int, default=3)
ap.add_argument("--iters", type=int, default=6)
a = ap.parse_args()
B, N, H, p = {"vitl": (8, 577, 16, 0.0), "c3p0": (32, 197, 12, 0.0), "c3p05": (32, 197, 12, 0.5), "c3p08": (32, 197, 12, 0.8), "n1024": (8, 1024, 12, 0.5)}[a.case]
dev = torch.device("cuda")
q, k, v, keep = synth.make_inputs(B, N, H, p, "random", "bf16", seed=0)
kb = keep.bool()
idx = torch.nonzero(kb.flatten()).flatten()
T = idx.numel()
def pk(t):
    out = torch.zeros(B * N, H, 64, dtype=t.dtype)
    out[:T] = t.reshape(B * N, H, 64)[idx]
    return out.to(dev)
cu = torch.zeros(B + 1, dtype=torch.int32)
cu[1:] = torch.cumsum(kb.sum(1), 0)
qp, kp, vp, cu = pk(q), pk(k), pk(v), cu.to(dev)
for _ in range(a.iters):
    rb.attn(qp, kp, vp, cu, N, engine=a.engine)
torch.cuda.synchronize()
print("ok")
