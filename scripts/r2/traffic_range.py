"""DRAM traffic of the fused C3 call over a WINDOW of launches (write-back
included): 16 rotating input/output sets, the calls between
cudaProfilerStart/Stop; run under
  ncu --replay-mode range --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
and divide by the launch count (printed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2604_15408_b200 as rb
import synth
B, N, H = 32, 197, 12
q, k, v, keep = synth.make_inputs(B, N, H, 0.8, "l2", "bf16", seed=0)
dev = torch.device("cuda")
sets = [dict(q=q.to(dev), k=k.to(dev), v=v.to(dev), keep=keep.to(dev),
             o=torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev),
             cu=torch.empty(B + 1, dtype=torch.int32, device=dev)) for _ in range(16)]
T = int(keep.numpy().astype(bool).sum())
for i in range(32):
    s = sets[i % 16]
    rb.pack_attend_unpack(s["q"], s["k"], s["v"], s["keep"], o=s["o"], cu=s["cu"], n_hint=T // B)
torch.cuda.synchronize()
L = 64
torch.cuda.profiler.start()
for i in range(L):
    s = sets[i % 16]
    rb.pack_attend_unpack(s["q"], s["k"], s["v"], s["keep"], o=s["o"], cu=s["cu"], n_hint=T // B)
torch.cuda.profiler.stop()
torch.cuda.synchronize()
print("launches", L)
