"""C3 fused time under a given RAGGED_LIB (occupancy experiments)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, bench, synth
import paper_2604_15408_b200 as rb
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
B, N, H = 32, 197, 12
q, k, v, keep = synth.make_inputs(B, N, H, 0.8, "l2", "bf16", seed=0)
sets = [dict(q=q.to(dev), k=k.to(dev), v=v.to(dev), keep=keep.to(dev), o=torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev),
             cu=torch.empty(B + 1, dtype=torch.int32, device=dev)) for _ in range(16)]
fn = [(lambda s=s: rb.pack_attend_unpack(s["q"], s["k"], s["v"], s["keep"], o=s["o"], cu=s["cu"], n_hint=39)) for s in sets]
r = {"lib": os.environ.get("RAGGED_LIB", "default")}
r["c3_us_2000"] = bench._graph_time(torch, fn, 2000)
r["c3_us_20"] = bench._graph_time(torch, fn, 20)
print(json.dumps(r))
