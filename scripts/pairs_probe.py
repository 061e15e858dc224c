"""clock64 probe of the tcgen05 pair path at p = 0 (needs libragged_tl.so).
Slots (slot 0, thread 0, first pass of its first problem): 0 pass start;
1 + 6j + 3X: S_X(j) ready; 2 + 6j + 3X: warp 0's P stored; 3 + 6j + 3X:
PV_X(j) + S_X(j+1) issued; 25 last commit seen; 26 pass 0 stored; 27 pass 1 stored."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RAGGED_LIB", os.path.join(ROOT, "paper_2604_15408_b200", "libragged_tl.so"))
import numpy as np, torch
import paper_2604_15408_b200 as rb, synth
p = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
B, N, H = 32, 197, 12
q, k, v, keep = (t.cuda() for t in synth.make_inputs(B, N, H, p, "l2", "bf16", seed=0))
o = torch.empty(B, N, H, 64, dtype=q.dtype, device="cuda")
for _ in range(3):
    rb.pack_attend_unpack(q, k, v, keep, o=o, engine=2)
torch.cuda.synchronize()
lib = rb.lib()
lib.ragged_debug_pairs_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
buf = np.zeros((148, 32), np.uint64)
lib.ragged_debug_pairs_timeline(buf.ctypes.data, 148)
t = buf.astype(np.int64)
t = t[t[:, 0] != 0]
rel = t - t[:, :1]
names = {0: "start"}
for j in range(4):
    for X in range(2):
        names[1 + 6 * j + 3 * X] = f"S{X}({j}) ready"
        names[2 + 6 * j + 3 * X] = f"P{X}({j}) stored"
        names[3 + 6 * j + 3 * X] = f"PV{X}({j}) issued"
names[25] = "last commit"; names[26] = "pass0 stored"; names[27] = "pass1 stored"
out = {}
for i in sorted(names):
    col = rel[:, i]
    col = col[col >= 0]
    out[names[i]] = [int(np.percentile(col, 50)), int(np.percentile(col, 90))] if len(col) else None
print(json.dumps(out, indent=1))
