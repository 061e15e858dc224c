"""Time the WS engine (ViT-L, C3 p0) under a given RAGGED_LIB build."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
res = {"lib": os.environ.get("RAGGED_LIB", "default")}
for name, B, N, H, p in (("vitl", 8, 577, 16, 0.0), ("c3p0", 32, 197, 12, 0.0)):
    sets = []
    for i in range(8):
        q, k, v, keep = synth.make_inputs(B, N, H, p, "random", "bf16", seed=i)
        kb = keep.bool(); idx = torch.nonzero(kb.flatten()).flatten(); T = idx.numel()
        def pk(t):
            out = torch.zeros(B * N, H, 64, dtype=t.dtype); out[:T] = t.reshape(B * N, H, 64)[idx]; return out.to(dev)
        cu = torch.zeros(B + 1, dtype=torch.int32); cu[1:] = torch.cumsum(kb.sum(1), 0)
        qp = pk(q); sets.append((qp, pk(k), pk(v), cu.to(dev), torch.empty_like(qp)))
    res[name] = bench._graph_time(torch, [(lambda s=s: rb.attn(s[0], s[1], s[2], s[3], N, op=s[4], engine=3)) for s in sets], 200)
print(json.dumps(res))
