import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2604_15408_b200 as rb, synth, oracle
DEV = "cuda"
B, N, H = 9, 197, 12
q, k, v, keep = [t.to(DEV) for t in synth.make_inputs(B, N, H, 0.7, "l2", "bf16", seed=3)]
keep[4, 0] = 0
keep[6] = 0
ref, rcu = rb.pack_attend_unpack(q, k, v, keep, want_cu=True)
o = torch.full((B, N, H, 64), -7.0, dtype=q.dtype, device=DEV)
cls = torch.full((B, H * 64), -7.0, dtype=q.dtype, device=DEV)
cu = torch.empty(B + 1, dtype=torch.int32, device=DEV)
rb.pack_attend_unpack_gather(q, k, v, keep, rb.gather_desc(1, 0, out=[o], cls=[cls]), cu=cu)
torch.cuda.synchronize()
d = (ref.view(torch.int16) != o.view(torch.int16)).any(-1).cpu().numpy()
bad = np.argwhere(d)
print("mismatching (b, n, h):", len(bad), bad[:20].tolist())
kn = keep.cpu().numpy()
for b_, n_, h_ in bad[:10]:
    print(b_, n_, h_, "kept" if kn[b_, n_] else "dropped", ref[b_, n_, h_, :4].tolist(), o[b_, n_, h_, :4].tolist())
g, _ = oracle.pack_attend_unpack(q.cpu(), k.cpu(), v.cpu(), kn)
print("cu", rcu.tolist(), cu.tolist())
print("ref err", float(np.abs(ref.double().cpu().numpy() - g).max()), "gather err", float(np.abs(o.double().cpu().numpy() - g).max()))
