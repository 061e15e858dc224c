"""LayerNorm A/B at the block's shapes (T live of B*N capacity rows), no hint (full grid)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
res = {"lib": os.environ.get("RAGGED_LIB", "default")}
D = 768
for T, cap in ((1248, 6304), (6304, 6304)):
    xs = [torch.randn(cap, D, device=dev).bfloat16() for _ in range(4)]
    w = torch.ones(D, device=dev).bfloat16(); b = torch.zeros(D, device=dev).bfloat16()
    y = torch.empty(cap, D, device=dev).bfloat16()
    live = torch.tensor([T], dtype=torch.int32, device=dev)
    res[f"T{T}_cap{cap}"] = bench._graph_time(torch, [(lambda x=x: rb.layer_norm(x, w, b, y=y, live=live)) for x in xs], 400)
print(json.dumps(res))
