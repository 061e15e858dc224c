"""Per-item clock64 timeline of the warp-specialised engine (TL build): for a
few CTAs, every item's Q issue, S_A(0) issue, softmax S-ready / P-stored per
block and tile, PV issue and epilogue, in us from the CTA's entry (1.965 GHz)."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("RAGGED_LIB", os.path.join(ROOT, "paper_2604_15408_b200", "libragged_tl.so"))
import numpy as np
import torch
import paper_2604_15408_b200 as rb
case = os.environ.get("CASE", "c3p0")
sys.argv = [sys.argv[0], "--case", case, "--iters", "3"]
if os.environ.get("FUSED"):
    import synth
    B, N, H, p = {"c3p0": (32, 197, 12, 0.0), "c3p05": (32, 197, 12, 0.5), "c3p08": (32, 197, 12, 0.8)}[case]
    q, k, v, keep = (x.cuda() for x in synth.make_inputs(B, N, H, p, "random", "bf16", seed=0))
    for _ in range(3):
        rb.pack_attend_unpack(q, k, v, keep, engine=3)
    torch.cuda.synchronize()
else:
    exec(open(os.path.join(ROOT, "scripts", "r2", "ws_one.py")).read().replace('print("ok")', ''))
lib = rb.lib()
lib.ragged_debug_fa_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
buf = np.zeros((148, 128), np.uint64)
lib.ragged_debug_fa_timeline(buf.ctypes.data, 148)
t = buf.astype(np.int64)
f = 1.0 / 1965.0
res = {"case": case}
for c in (0, 1, 60, 147):
    base = t[c, 48]
    us = lambda s: round((t[c, s] - base) * f, 3) if t[c, s] else None
    r = {"end": us(58), "first_SA": us(49),
         "sm_inner_first": {k: us(64 + i) for i, k in enumerate(("pass1_loaded", "max_done", "chunk0", "chunk3", "chunk7"))}}
    for it in range(4):
        r[f"item{it}"] = {"Q_issue": us(59 + it), "SA0_issue": us(32 + 4 * it + 3), "PA0_seen": us(32 + 4 * it),
                          "PVA0_issued": us(33 + 4 * it),
                          "A": [(us(4 * it + 2 * j), us(4 * it + 2 * j + 1)) for j in range(2)],
                          "B": [(us(16 + 4 * it + 2 * j), us(16 + 4 * it + 2 * j + 1)) for j in range(2)],
                          "epiA": us(50 + it), "epiB": us(54 + it), "rows_pub": us(70 + it), "kv_last_issue": us(74 + it)}
    res[f"cta{c}"] = r
print(json.dumps(res, indent=1))
