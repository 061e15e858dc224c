"""clock64 probe of the mma.sync fused kernel (TL build): thread 0 of each CTA,
0 = gathers landed, 1 = first chunk's S + row max done, 2 = first slice's O
staged; with the %globaltimer timeline of the same launch -> effective clock."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RAGGED_LIB", os.path.join(ROOT, "paper_2604_15408_b200", "libragged_tl.so"))
import numpy as np, torch
import paper_2604_15408_b200 as rb, synth
B, N, H = 32, 197, 12
q, k, v, keep = (t.cuda() for t in synth.make_inputs(B, N, H, 0.8, "l2", "bf16", seed=0))
o = torch.empty(B, N, H, 64, dtype=q.dtype, device="cuda")
for _ in range(20):
    rb.pack_attend_unpack(q, k, v, keep, o=o, engine=1)
torch.cuda.synchronize()
lib = rb.lib()
lib.ragged_debug_pairs_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
lib.ragged_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
n = B * H
pc = np.zeros((n, 32), np.uint64); lib.ragged_debug_pairs_timeline(pc.ctypes.data, n)
tl = np.zeros((n, 16), np.uint64); lib.ragged_debug_timeline(tl.ctypes.data, n)
pc = pc.astype(np.int64); tl = tl.astype(np.int64)
ok = (pc[:, 0] != 0) & (pc[:, 2] != 0)
cyc_qk = pc[ok, 1] - pc[ok, 0]
cyc_slice = pc[ok, 2] - pc[ok, 0]
ns_slice = tl[ok, 6] - tl[ok, 3]
print(json.dumps({"cycles_gathers_to_first_rowmax": [int(np.percentile(cyc_qk, q)) for q in (50, 90)],
                  "cycles_gathers_to_O_staged": [int(np.percentile(cyc_slice, q)) for q in (50, 90)],
                  "ns_gathers_to_O_staged": [int(np.percentile(ns_slice, q)) for q in (50, 90)],
                  "effective_GHz": float(np.median(cyc_slice / np.maximum(ns_slice, 1)))}))
