"""Time ragged_linear at the N1 block's small-T shapes (B=32, p=0.8: T=1248 live
of 6304 capacity rows) under the process's RAGGED_GEMM_SPLIT setting."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, bench
import paper_2604_15408_b200 as rb
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
res = {"split_env": os.environ.get("RAGGED_GEMM_SPLIT", "auto")}
T = 1248
for name, N, K, epi in (("qkv", 2304, 768, 0), ("proj", 768, 768, 2), ("fc1", 3072, 768, 1), ("fc2", 768, 3072, 2)):
    g = torch.Generator().manual_seed(1)
    a = torch.randn(T, K, generator=g).bfloat16().to(dev)
    w = (0.05 * torch.randn(N, K, generator=g)).bfloat16().to(dev)
    b = torch.zeros(N, dtype=torch.bfloat16, device=dev)
    r = torch.randn(T, N, generator=g).bfloat16().to(dev) if epi == 2 else None
    o = torch.empty(T, N, dtype=torch.bfloat16, device=dev)
    res[name] = bench._graph_time(torch, [lambda: rb.linear(a, w, b, epi, r, out=o)], 200)
print(json.dumps(res))
