"""One C3 (H = 12) prune-fused call after warm-up, for ncu source-level capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda")
B, N, H = 32, 197, 12
kk = synth.kept_tokens(N, 0.8)
x = synth.hidden_states(B, N, H * 64, "bf16", seed=40).to(dev)
q, k, v = (t.to(dev) for t in synth.activations(B, N, H, 64, "bf16", seed=90))
o = torch.empty_like(q)
for _ in range(4):
    rb.prune_l2_pack_attend_unpack(x, q, k, v, kk, o=o)
torch.cuda.synchronize()
print("ok")
