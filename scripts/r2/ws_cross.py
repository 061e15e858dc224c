"""WS engine vs mma.sync over DeiT/ViT-L lengths (crossover for AUTO), with the
max-abs error vs the fp64 oracle on a sampled image set; RAGGED_LIB selects a build."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import bench
import oracle
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
res = {"lib": os.environ.get("RAGGED_LIB", "default")}
cases = [("C3_p0", 32, 197, 12, 0.0), ("C3_p0.2", 32, 197, 12, 0.2), ("C3_p0.3", 32, 197, 12, 0.3),
         ("C3_p0.4", 32, 197, 12, 0.4), ("C3_p0.5", 32, 197, 12, 0.5), ("C3_p0.8", 32, 197, 12, 0.8),
         ("vitl", 8, 577, 16, 0.0), ("N1024_p0.5", 8, 1024, 12, 0.5)]
for name, B, N, H, p in cases:
    kk = synth.kept_tokens(N, p)
    sets = []
    for i in range(8):
        for dist in (["standard", "peaked"] if i == 0 else ["standard"]):
            q, k, v, keep = synth.make_inputs(B, N, H, p, "random", "bf16", seed=i)
            if dist == "peaked":
                q, k, v = synth.activations(B, N, H, 64, torch.bfloat16, 77, "peaked")
            kb = keep.bool(); idx = torch.nonzero(kb.flatten()).flatten(); T = idx.numel()
            def pk(t):
                out = torch.zeros(B * N, H, 64, dtype=t.dtype); out[:T] = t.reshape(B * N, H, 64)[idx]; return out
            cu = torch.zeros(B + 1, dtype=torch.int32); cu[1:] = torch.cumsum(kb.sum(1), 0)
            host = (pk(q), pk(k), pk(v), cu)
            sets.append(dict(host=host, dist=dist, T=T, d=(host[0].to(dev), host[1].to(dev), host[2].to(dev), cu.to(dev),
                                                       torch.empty(B * N, H, 64, dtype=torch.bfloat16, device=dev))))
    r = {"n": kk}
    for eng, nm in ((3, "ws"), (1, "mma")):
        r[nm + "_us"] = bench._graph_time(torch, [(lambda s=s["d"], e=eng: rb.attn(s[0], s[1], s[2], s[3], N, op=s[4], engine=e, n_hint=kk)) for s in sets], 200)
    # accuracy of the WS engine on the first two sets (standard, peaked), 4 images
    for s in sets[:2]:
        qh, kh, vh, cu = s["host"]
        nb = 4
        T4 = int(cu[nb])
        out = rb.attn(*s["d"][:4], N, engine=3)
        torch.cuda.synchronize()
        got = out[:T4].double().cpu().numpy()
        ref = oracle.attention(qh[:T4], kh[:T4], vh[:T4], cu[:nb + 1].numpy())
        r["err_" + s["dist"]] = float(np.abs(got - ref).max())
    res[name] = r
    print(name, r, flush=True)
print(json.dumps(res))
