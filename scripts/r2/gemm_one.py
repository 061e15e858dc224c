"""Run one ragged_linear shape a few times (for ncu):  python gemm_one.py T N K epi"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_15408_b200 as rb
T, N, K, epi = [int(x) for x in sys.argv[1:5]]
dev = torch.device("cuda", 0)
g = torch.Generator().manual_seed(1)
a = torch.randn(T, K, generator=g).bfloat16().to(dev)
w = (0.05 * torch.randn(N, K, generator=g)).bfloat16().to(dev)
b = torch.zeros(N, dtype=torch.bfloat16, device=dev)
r = torch.randn(T, N, generator=g).bfloat16().to(dev) if epi == 2 else None
o = torch.empty(T, N, dtype=torch.bfloat16, device=dev)
for _ in range(4):
    rb.linear(a, w, b, epi, r, out=o)
torch.cuda.synchronize()
