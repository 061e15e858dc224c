"""Fused pack-attend-unpack on the warp-specialised engine (gather4): correctness vs the
fp64 oracle and the mma.sync fused path, cu_seqlens, +0.0 rows; timing vs the mma.sync
fused kernel over the C3 sweep and C2/C4 shapes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import bench
import oracle
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
res = {"check": {}, "time": {}}
# correctness
for (B, N, H, p, m) in [(3, 197, 2, 0.0, "all"), (4, 197, 3, 0.5, "l2"), (5, 197, 2, 0.2, "random"), (3, 256, 2, 0.3, "ats"),
                        (2, 33, 4, 0.5, "random"), (6, 197, 12, 0.8, "l2"), (2, 1, 2, 0.0, "all")]:
    q, k, v, keep = synth.make_inputs(B, N, H, p, m, "bf16", seed=B + N)
    keep = keep.clone()
    if B > 2:
        keep[1] = 0  # an empty image
    qd, kd, vd, kpd = (t.to(dev) for t in (q, k, v, keep))
    o = torch.full((B, N, H, 64), 7.0, dtype=torch.bfloat16, device=dev)
    cu = torch.full((B + 1,), -5, dtype=torch.int32, device=dev)
    rb.pack_attend_unpack(qd, kd, vd, kpd, o=o, cu=cu, engine=3)
    om, cum = rb.pack_attend_unpack(qd, kd, vd, kpd, want_cu=True, engine=1)
    torch.cuda.synchronize()
    ref, rcu = oracle.pack_attend_unpack(q, k, v, keep.numpy())
    err = float(np.abs(o.double().cpu().numpy() - ref).max())
    kb = keep.numpy().astype(bool)
    zeros_ok = bool((o.cpu().view(torch.int16).numpy()[~kb] == 0).all())
    res["check"][f"B{B}_N{N}_H{H}_p{p}_{m}"] = {"err": err, "cu_ok": cu.cpu().tolist() == rcu.tolist(), "zeros_ok": zeros_ok,
                                                "err_mma": float(np.abs(om.double().cpu().numpy() - ref).max())}
    print(res["check"][f"B{B}_N{N}_H{H}_p{p}_{m}"], flush=True)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
for (B, N, H) in [(32, 197, 12), (32, 197, 6), (64, 197, 12)]:
    for p in (0.0, 0.1, 0.2, 0.3, 0.5):
        kk = synth.kept_tokens(N, p)
        sets = []
        for i in range(16):
            q, k, v, keep = synth.make_inputs(B, N, H, p, "l2", "bf16", seed=i)
            sets.append(dict(q=q.to(dev), k=k.to(dev), v=v.to(dev), keep=keep.to(dev),
                             o=torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev),
                             cu=torch.empty(B + 1, dtype=torch.int32, device=dev)))
        r = {}
        for eng, nm in ((3, "ws"), (1, "mma")):
            r[nm + "_us"] = bench._graph_time(torch, [(lambda s=s, e=eng: rb.pack_attend_unpack(
                s["q"], s["k"], s["v"], s["keep"], o=s["o"], cu=s["cu"], engine=e, n_hint=kk)) for s in sets], 200)
        res["time"][f"B{B}_H{H}_p{p}"] = r
        print(B, H, p, r, flush=True)
print(json.dumps(res))
