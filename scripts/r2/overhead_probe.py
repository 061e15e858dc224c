"""Where does the fixed per-replay cost of bench.py's K-step graph go?
Times the C3 fused call as bench.py does (K steps in one graph, 16 cold sets)
for K in {1, 5, 20, 200, 2000}, with and without a gate kernel (torch.cuda._sleep)
queued ahead of the start event so that the host's graph submission is off the
device clock."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_15408_b200 as rb
import synth

dev = torch.device("cuda", 0)
B, N, H = 32, 197, 12
q, k, v, keep = synth.make_inputs(B, N, H, 0.8, "l2", "bf16", seed=0)
T = int(keep.numpy().astype(bool).sum())
sets = [dict(q=q.to(dev), k=k.to(dev), v=v.to(dev), keep=keep.to(dev),
             o=torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev),
             cu=torch.empty(B + 1, dtype=torch.int32, device=dev)) for _ in range(16)]

def step(i):
    s = sets[i % 16]
    rb.pack_attend_unpack(s["q"], s["k"], s["v"], s["keep"], o=s["o"], cu=s["cu"], n_hint=T // B)

for i in range(20):
    step(i)
torch.cuda.synchronize()
res = {}
for K in (1, 5, 20, 200, 2000):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        for i in range(K):
            step(i)
    g.replay(); torch.cuda.synchronize()
    for gate in (False, True):
        ts = []
        for rep in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            if gate:
                torch.cuda._sleep(200000)
            a.record(); g.replay(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / K)
        ts.sort()
        res[f"K{K}_{'gate' if gate else 'nogate'}"] = {"median_us_per_call": ts[3], "min": ts[0]}
print(json.dumps(res, indent=1))
