"""Fused prune timing vs cluster size H (B*H = 384 CTAs in every case)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
N = 197
res = {}
for B, H in ((128, 3), (64, 6), (48, 8), (32, 12), (24, 16)):
    kk = synth.kept_tokens(N, 0.8)
    sets = []
    for i in range(8):
        x = synth.hidden_states(B, N, H * 64, "bf16", seed=70 + i).to(dev)
        q, k, v = (t.to(dev) for t in synth.activations(B, N, H, 64, "bf16", seed=80 + i))
        keep = torch.from_numpy(synth.mask_threshold_l2(B, N, kk, seed=3, D=H * 64)).to(dev)
        sets.append(dict(x=x, q=q, k=k, v=v, keep=keep, o=torch.empty_like(q)))
    res[f"B{B}_H{H}_prune_fused_us"] = bench._graph_time(torch, [(lambda s=s: rb.prune_l2_pack_attend_unpack(
        s["x"], s["q"], s["k"], s["v"], kk, o=s["o"])) for s in sets], 300)
    res[f"B{B}_H{H}_fused_only_us"] = bench._graph_time(torch, [(lambda s=s: rb.pack_attend_unpack(
        s["q"], s["k"], s["v"], s["keep"], o=s["o"], n_hint=kk)) for s in sets], 300)
    del sets
print(json.dumps(res, indent=1))
