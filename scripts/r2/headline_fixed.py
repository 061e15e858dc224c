"""Fixed per-region cost of the headline timing: K fused C3 calls after the
device gate, (a) captured in one CUDA graph, (b) launched eagerly on the stream
(the host enqueues them while the gate spins).  us per call for several K."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
B, N, H, p = 32, 197, 12, 0.8
q, k, v, keep = synth.make_inputs(B, N, H, p, "l2", "bf16", seed=0)
T = int(keep.sum())
sets = [dict(q=q.to(dev), k=k.to(dev), v=v.to(dev), keep=keep.to(dev), o=torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev),
             cu=torch.empty(B + 1, dtype=torch.int32, device=dev)) for _ in range(bench.N_SETS)]
def step(i):
    s = sets[i % len(sets)]
    rb.pack_attend_unpack(s["q"], s["k"], s["v"], s["keep"], o=s["o"], cu=s["cu"], n_hint=T // B)
for i in range(10): step(i)
torch.cuda.synchronize()
stream = torch.cuda.current_stream()
res = {}
for K in (1, 2, 5, 10, 20, 50, 200):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        for i in range(K): step(i)
    torch.cuda.synchronize(); g.replay(); torch.cuda.synchronize()
    tg, te = [], []
    for rep in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(bench.GATE_CYCLES); a.record(stream); g.replay(); b.record(stream); torch.cuda.synchronize()
        tg.append(1e3 * a.elapsed_time(b) / K)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(bench.GATE_CYCLES); a.record(stream)
        for i in range(K): step(i)
        b.record(stream); torch.cuda.synchronize()
        te.append(1e3 * a.elapsed_time(b) / K)
    res[K] = {"graph_us": statistics.median(tg), "eager_us": statistics.median(te)}
    print(K, res[K], flush=True)
print(json.dumps(res))
