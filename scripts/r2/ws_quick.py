"""Timing of the warp-specialised engine vs the mma.sync kernels and FA2 varlen."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import bench
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
res = {}
cases = [("C3_p0_B32_N197_H12", 32, 197, 12, 0.0), ("C3_p0.5", 32, 197, 12, 0.5), ("C3_p0.8", 32, 197, 12, 0.8),
         ("vitl_N577_B8_H16_p0", 8, 577, 16, 0.0), ("N1024_B8_H12_p0.5", 8, 1024, 12, 0.5),
         ("vitl_N577_p0.7", 8, 577, 16, 0.7)]
for name, B, N, H, p in cases:
    kk = synth.kept_tokens(N, p)
    sets = []
    for i in range(8):
        q, k, v, keep = synth.make_inputs(B, N, H, p, "random", "bf16", seed=i)
        kb = keep.bool()
        idx = torch.nonzero(kb.flatten()).flatten()
        T = idx.numel()
        def pk(t):
            out = torch.zeros(B * N, H, 64, dtype=t.dtype)
            out[:T] = t.reshape(B * N, H, 64)[idx]
            return out.to(dev)
        cu = torch.zeros(B + 1, dtype=torch.int32)
        cu[1:] = torch.cumsum(kb.sum(1), 0)
        qp = pk(q)
        sets.append((qp, pk(k), pk(v), cu.to(dev), torch.empty_like(qp)))
    torch.cuda.synchronize()
    r = {"T": int(sets[0][3][-1].item())}
    for eng, nm in ((3, "ws"), (2, "tc"), (1, "mma"), (0, "auto")):
        try:
            r[nm + "_us"] = bench._graph_time(torch, [(lambda s=s, e=eng: rb.attn(s[0], s[1], s[2], s[3], N, op=s[4], engine=e, n_hint=kk)) for s in sets], 200)
        except Exception as ex:
            r[nm + "_us"] = repr(ex)[:100]
    try:
        from flash_attn import flash_attn_varlen_func
        T = r["T"]
        fa = [(lambda s=s: flash_attn_varlen_func(s[0][:T], s[1][:T], s[2][:T], s[3], s[3], kk, kk)) for s in sets]
        r["fa2_us"] = bench._graph_time(torch, fa, 200)
    except Exception as ex:
        r["fa2_us"] = repr(ex)[:100]
    n = kk
    r["flops"] = 4 * B * H * n * n * 64
    if isinstance(r["ws_us"], float):
        r["ws_tflops"] = r["flops"] / (r["ws_us"] * 1e-6) / 1e12
    res[name] = r
    print(name, r, flush=True)
print(json.dumps(res))

# the fused path per engine (C3 shapes, padded inputs)
for p in (0.0, 0.5, 0.8):
    B, N, H = 32, 197, 12
    kk = synth.kept_tokens(N, p)
    sets = []
    for i in range(8):
        q, k, v, keep = synth.make_inputs(B, N, H, p, "random", "bf16", seed=i)
        sets.append((q.to(dev), k.to(dev), v.to(dev), keep.to(dev), torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev)))
    r = {}
    for eng, nm in ((2, "tc"), (1, "mma"), (0, "auto")):
        try:
            r[nm + "_us"] = bench._graph_time(torch, [(lambda s=s, e=eng: rb.pack_attend_unpack(s[0], s[1], s[2], s[3], o=s[4], engine=e, n_hint=kk)) for s in sets], 200)
        except Exception as ex:
            r[nm + "_us"] = repr(ex)[:100]
    print(f"fused_C3_p{p}", r, flush=True)
