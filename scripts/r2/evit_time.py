"""EViT keep mask (+ fused token) at C3 and C4 shapes, alone and ahead of the fused path."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
res = {}
for B, H, p in ((32, 12, 0.8), (64, 12, 0.7), (32, 6, 0.5)):
    N = 197
    kk = synth.kept_tokens(N, p)
    ev = []
    for i in range(16):
        q, k, v = (t.to(dev) for t in synth.activations(B, N, H, 64, "bf16", seed=i))
        ev.append(dict(q=q, k=k, v=v, keep=torch.empty(B, N, dtype=torch.uint8, device=dev),
                       o=torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev)))
    r = {"mask_us": bench._graph_time(torch, [(lambda e=e: rb.keep_evit(e["q"], e["k"], e["v"], kk, keep=e["keep"])) for e in ev], 200)}
    def ef(e):
        rb.keep_evit(e["q"], e["k"], e["v"], kk, keep=e["keep"])
        rb.pack_attend_unpack(e["q"], e["k"], e["v"], e["keep"], o=e["o"], n_hint=kk)
    r["mask_then_fused_us"] = bench._graph_time(torch, [(lambda e=e: ef(e)) for e in ev], 200)
    res[f"B{B}_H{H}_p{p}"] = r
    print(B, H, p, r, flush=True)
print(json.dumps(res))
