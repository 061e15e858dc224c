"""N2 Threshold-l2 mask at C3: cluster kernel vs the row-parallel workspace kernel,
alone and ahead of the fused path (graph replay, 17 rotating hidden-state batches)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
res = {}
for B, N, H, p in ((32, 197, 12, 0.8), (64, 197, 12, 0.7), (4096, 197, 12, 0.7)):
    NX = 17 if B <= 64 else 3
    xs = [synth.hidden_states(B, N, H * 64, "bf16", seed=40 + i).to(dev) for i in range(NX)]
    kk = synth.kept_tokens(N, p)
    nk = 16 if B <= 64 else 2
    keeps = [torch.empty(B, N, dtype=torch.uint8, device=dev) for _ in range(nk)]
    q, k, v = (t.to(dev) for t in synth.activations(B, N, H, 64, "bf16", seed=1))
    o = torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev)
    ws = rb.l2_workspace(B, N, dev)
    L = NX * nk
    reps = 200 if B <= 64 else 20
    r = {}
    r["cluster_us"] = bench._graph_time(torch, [(lambda j=j: rb.keep_topk_l2(xs[j % NX], kk, keep=keeps[j % nk])) for j in range(L)], reps)
    r["ws_us"] = bench._graph_time(torch, [(lambda j=j: rb.keep_topk_l2(xs[j % NX], kk, keep=keeps[j % nk], workspace=ws)) for j in range(L)], reps)
    def pf(j, w):
        rb.keep_topk_l2(xs[j % NX], kk, keep=keeps[j % nk], workspace=w)
        rb.pack_attend_unpack(q, k, v, keeps[j % nk], o=o, n_hint=kk)
    r["cluster_then_fused_us"] = bench._graph_time(torch, [(lambda j=j: pf(j, None)) for j in range(L)], reps)
    r["ws_then_fused_us"] = bench._graph_time(torch, [(lambda j=j: pf(j, ws)) for j in range(L)], reps)
    r["fused_alone_us"] = bench._graph_time(torch, [(lambda j=j: rb.pack_attend_unpack(q, k, v, keeps[j % nk], o=o, n_hint=kk)) for j in range(L)], reps)
    byts = B * N * H * 128 + B * N
    r["ws_hbm_frac"] = byts / (r["ws_us"] * 1e-6) / 1e9 / bench._hbm_peak()
    res[f"B{B}_p{p}"] = r
    print(B, r, flush=True)
print(json.dumps(res))
