"""Quick N2 timing: l2 mask, EViT mask, mask -> fused at C3 (bench.py's helpers)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
import synth

dev = torch.device("cuda", 0)
B, N, H = 32, 197, 12
q, k, v, keep = synth.make_inputs(B, N, H, 0.8, "l2", "bf16", seed=0)
sets = [dict(q=q.to(dev), k=k.to(dev), v=v.to(dev), keep=keep.to(dev),
             o=torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev),
             cu=torch.empty(B + 1, dtype=torch.int32, device=dev)) for _ in range(bench.N_SETS)]
kk = synth.kept_tokens(N, 0.8)
res = {"fused_us": bench._graph_time(torch, [(lambda s=s: rb.pack_attend_unpack(s["q"], s["k"], s["v"], s["keep"], o=s["o"], cu=s["cu"], n_hint=kk)) for s in sets], 500)}
NX = 17
xs = [synth.hidden_states(B, N, H * 64, "bf16", seed=40 + i).to(dev) for i in range(NX)]
keeps = [torch.empty(B, N, dtype=torch.uint8, device=dev) for _ in range(16)]
L = 16 * NX
res["l2_us"] = bench._graph_time(torch, [(lambda j=j: rb.keep_topk_l2(xs[j % NX], kk, keep=keeps[j % 16])) for j in range(L)], 500)
def pf(j):
    s = sets[j % 16]
    rb.keep_topk_l2(xs[j % NX], kk, keep=keeps[j % 16])
    rb.pack_attend_unpack(s["q"], s["k"], s["v"], keeps[j % 16], o=s["o"], cu=s["cu"], n_hint=kk)
res["l2_then_fused_us"] = bench._graph_time(torch, [(lambda j=j: pf(j)) for j in range(L)], 500)
ev = [dict(q=s["q"].clone(), k=s["k"].clone(), v=s["v"].clone(), keep=torch.empty_like(s["keep"])) for s in sets]
res["evit_us"] = bench._graph_time(torch, [(lambda e=e: rb.keep_evit(e["q"], e["k"], e["v"], kk, keep=e["keep"])) for e in ev], 500)
def ef(i):
    e, s = ev[i], sets[i]
    rb.keep_evit(e["q"], e["k"], e["v"], kk, keep=e["keep"])
    rb.pack_attend_unpack(e["q"], e["k"], e["v"], e["keep"], o=s["o"], cu=s["cu"], n_hint=kk)
res["evit_then_fused_us"] = bench._graph_time(torch, [(lambda i=i: ef(i)) for i in range(16)], 500)
res["l2_hbm_frac"] = (B * N * H * 128 + B * N) / (res["l2_us"] * 1e-6) / 1e9 / bench._hbm_peak()
print(json.dumps(res, indent=1))
pr = []
for j in range(L):
    pass
def fp(j):
    s = sets[j % 16]
    rb.prune_l2_pack_attend_unpack(xs[j % NX], s["q"], s["k"], s["v"], kk, o=s["o"], cu=s["cu"])
res["prune_l2_fused_us"] = bench._graph_time(torch, [(lambda j=j: fp(j)) for j in range(L)], 500)
print(json.dumps({"prune_l2_fused_us": res["prune_l2_fused_us"]}))
