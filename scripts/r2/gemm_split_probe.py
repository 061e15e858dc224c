"""Time ragged_linear at the N1 block's shapes (B=32: T=1248 live at p=0.8,
6304 at p=0) under the process's RAGGED_GEMM_SPLIT / RAGGED_GEMM_MCAST
settings, beside torch (cuBLAS) on the same operands."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, bench
import paper_2604_15408_b200 as rb
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
res = {"split_env": os.environ.get("RAGGED_GEMM_SPLIT", "auto"), "mcast_env": os.environ.get("RAGGED_GEMM_MCAST", "auto")}
for T in [int(t) for t in os.environ.get("PROBE_T", "1248").split(",")]:
    for name, N, K, epi in (("qkv", 2304, 768, 0), ("proj", 768, 768, 2), ("fc1", 3072, 768, 1), ("fc2", 768, 3072, 2)):
        g = torch.Generator().manual_seed(1)
        a = torch.randn(T, K, generator=g).bfloat16().to(dev)
        w = (0.05 * torch.randn(N, K, generator=g)).bfloat16().to(dev)
        b = torch.zeros(N, dtype=torch.bfloat16, device=dev)
        r = torch.randn(T, N, generator=g).bfloat16().to(dev) if epi == 2 else None
        o = torch.empty(T, N, dtype=torch.bfloat16, device=dev)
        ref = torch.nn.functional.linear(a.float(), w.float(), b.float())
        if epi == 1: ref = torch.nn.functional.gelu(ref)
        if epi == 2: ref = ref + r.float()
        rb.linear(a, w, b, epi, r, out=o); torch.cuda.synchronize()
        err = float((o.float() - ref).abs().max())
        ours = bench._graph_time(torch, [lambda: rb.linear(a, w, b, epi, r, out=o)], 200)
        if epi == 2:
            cub = bench._graph_time(torch, [lambda: torch.addmm(r, a, w.t(), out=o)], 200)
        else:
            cub = bench._graph_time(torch, [lambda: torch.addmm(b, a, w.t(), out=o)], 200)
        res[f"{name}_T{T}"] = {"ours_us": ours, "cublas_us": cub, "max_err": err}
print(json.dumps(res))
