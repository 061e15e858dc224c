"""Where does the N2 mask kernel's time go?  hot vs cold inputs, early-exit EViT
(launch + grid-dependency floor of a cluster kernel), empty kernel."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
import synth

dev = torch.device("cuda", 0)
B, N, H = 32, 197, 12
kk = synth.kept_tokens(N, 0.8)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()   # clocks up
res = {}
for Bx in (32, 128, 512):
    xs = [synth.hidden_states(Bx, N, H * 64, "bf16", seed=40 + i).to(dev) for i in range(17 if Bx == 32 else 3)]
    keep = torch.empty(Bx, N, dtype=torch.uint8, device=dev)
    res[f"l2_B{Bx}_hot"] = bench._graph_time(torch, [lambda: rb.keep_topk_l2(xs[0], kk, keep=keep)], 500)
    res[f"l2_B{Bx}_cold"] = bench._graph_time(torch, [(lambda j=j: rb.keep_topk_l2(xs[j], kk, keep=keep)) for j in range(len(xs))], 500)
    res[f"l2_B{Bx}_cold_frac"] = (Bx * N * H * 128) / (res[f"l2_B{Bx}_cold"] * 1e-6) / 1e9 / bench._hbm_peak()
    del xs
q, k, v = (t.to(dev) for t in synth.activations(B, N, H, 64, "bf16", seed=1))
keep = torch.empty(B, N, dtype=torch.uint8, device=dev)
res["evit_allkeep_us"] = bench._graph_time(torch, [lambda: rb.keep_evit(q, k, v, N, keep=keep)], 500)
res["evit_k1_us"] = bench._graph_time(torch, [lambda: rb.keep_evit(q, k, v, 1, keep=keep)], 500)
res["evit_hot_us"] = bench._graph_time(torch, [lambda: rb.keep_evit(q, k, v, kk, keep=keep)], 500)
res["empty_256x256_us"] = bench._graph_time(torch, [lambda: rb.empty_launch(256, 256)], 500)
print(json.dumps(res, indent=1))
# mask -> fused (two launches) vs the single-launch prune kernel, H = 12 and 6
for Hh in (12, 6):
    xs = [synth.hidden_states(B, N, Hh * 64, "bf16", seed=40 + i).to(dev) for i in range(17)]
    qs = [tuple(t.to(dev) for t in synth.activations(B, N, Hh, 64, "bf16", seed=90 + i)) for i in range(16)]
    o = torch.empty_like(qs[0][0])
    keeps = [torch.empty(B, N, dtype=torch.uint8, device=dev) for _ in range(16)]
    def two(j):
        rb.keep_topk_l2(xs[j % 17], kk, keep=keeps[j % 16])
        q_, k_, v_ = qs[j % 16]
        rb.pack_attend_unpack(q_, k_, v_, keeps[j % 16], o=o, n_hint=kk)
    def one(j):
        q_, k_, v_ = qs[j % 16]
        rb.prune_l2_pack_attend_unpack(xs[j % 17], q_, k_, v_, kk, o=o)
    def fused_only(j):
        q_, k_, v_ = qs[j % 16]
        rb.pack_attend_unpack(q_, k_, v_, keeps[j % 16], o=o, n_hint=kk)
    L = 16 * 17
    res[f"H{Hh}_mask_then_fused_us"] = bench._graph_time(torch, [(lambda j=j: two(j)) for j in range(L)], 500)
    res[f"H{Hh}_fused_only_us"] = bench._graph_time(torch, [(lambda j=j: fused_only(j)) for j in range(L)], 500)
    res[f"H{Hh}_prune_in_fused_us"] = bench._graph_time(torch, [(lambda j=j: one(j)) for j in range(L)], 500)
    del xs, qs
print(json.dumps(res, indent=1))
