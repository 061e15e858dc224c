"""clock64 timeline of the warp-specialised engine's first item per CTA (TL build)."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("RAGGED_LIB", os.path.join(ROOT, "paper_2604_15408_b200", "libragged_tl.so"))
sys.argv += [] 
import numpy as np
import torch
import paper_2604_15408_b200 as rb
sys.argv = [sys.argv[0], "--case", os.environ.get("CASE", "vitl"), "--iters", "3"]
exec(open(os.path.join(ROOT, "scripts", "r2", "ws_one.py")).read().replace('print("ok")', ''))
lib = rb.lib()
lib.ragged_debug_fa_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
buf = np.zeros((148, 128), np.uint64)
lib.ragged_debug_fa_timeline(buf.ctypes.data, 148)
t = buf.astype(np.int64)
res = {}
for c in (0, 1, 50, 100):
    base = t[c, 48]
    r = {k: int(t[c, s] - base) for k, s in (("first_SA_issue", 49), ("first_epi_A", 50), ("end", 51))}
    r["A_S_ready_P_done"] = [(int(t[c, 2 * j] - base), int(t[c, 2 * j + 1] - base)) for j in range(8) if t[c, 2 * j]]
    r["B_S_ready_P_done"] = [(int(t[c, 16 + 2 * j] - base), int(t[c, 17 + 2 * j] - base)) for j in range(8) if t[c, 16 + 2 * j]]
    r["MMA_PA_seen_issued"] = [(int(t[c, 32 + 2 * j] - base), int(t[c, 33 + 2 * j] - base)) for j in range(8) if t[c, 32 + 2 * j]]
    res[f"cta{c}"] = r
print(json.dumps(res, indent=1))
