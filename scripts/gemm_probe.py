"""GEMM phase probe (TL build): median/p90 over CTAs of the block.cu GT stamps,
relative to the earliest CTA entry (us).  python scripts/gemm_probe.py T N K epi"""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RAGGED_LIB", os.path.join(ROOT, "paper_2604_15408_b200", "libragged_tl.so"))
import numpy as np, torch
import paper_2604_15408_b200 as rb
T, N, K, epi = [int(x) for x in sys.argv[1:5]]
a = torch.randn(T, K, device="cuda").bfloat16(); w = (0.02 * torch.randn(N, K, device="cuda")).bfloat16()
r = torch.randn(T, N, device="cuda").bfloat16(); o = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    rb.linear(a, w, None, epi, r if epi == 2 else None, out=o)
torch.cuda.synchronize()
lib = rb.lib()
lib.ragged_debug_gemm_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
buf = np.zeros((1024, 8), np.uint64)
lib.ragged_debug_gemm_timeline(buf.ctypes.data, 1024)
t = buf.astype(np.int64)
t = t[(t[:, 0] != 0) & (t[:, 4] != 0)]
rel = (t - t[:, 0].min()) / 1e3
names = ["entry", "setup", "pdl_wait", "first_stage", "last_mma_issued", "acc_ready", "stored", "exit"]
print(json.dumps({f"{T}x{N}x{K}": {n: [round(float(np.percentile(rel[:, i], q)), 2) for q in (50, 90)]
                                   for i, n in enumerate(names)}, "ctas": int(len(t))}))
