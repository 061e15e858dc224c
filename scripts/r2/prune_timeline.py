"""Per-CTA phase timeline of the N2 mask kernels (TL build), back to back."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("RAGGED_LIB", os.path.join(ROOT, "paper_2604_15408_b200", "libragged_tl.so"))
import numpy as np
import torch
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda")
B, N, H = 32, 197, 12
kk = synth.kept_tokens(N, 0.8)
lib = rb.lib()
lib.ragged_debug_prune_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
xs = [synth.hidden_states(B, N, H * 64, "bf16", seed=40 + i).to(dev) for i in range(4)]
q, k, v = (t.to(dev) for t in synth.activations(B, N, H, 64, "bf16", seed=1))
keep = torch.empty(B, N, dtype=torch.uint8, device=dev)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()   # clocks up
res = {}
for name, fn in (("l2", lambda i: rb.keep_topk_l2(xs[i % 4], kk, keep=keep)),
                 ("evit", lambda i: rb.keep_evit(q, k, v, kk, keep=keep))):
    for mode in ("isolated", "back_to_back"):
        for i in range(8):
            fn(i)
        torch.cuda.synchronize()
        if mode == "isolated":
            fn(1)
        else:
            for i in range(8):
                fn(i)
        torch.cuda.synchronize()
        buf = np.zeros((B * 8, 16), np.uint64)
        lib.ragged_debug_prune_timeline(buf.ctypes.data, B * 8)
        t = buf.astype(np.int64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        nslot = 7 if name == "l2" else 12
        if name == "l2":
            sm = buf[:, 15].astype(np.int64)
            cnt = np.bincount(sm, minlength=148)
            res[f"{name}_{mode}_sm_use"] = {"distinct_sms": int((cnt > 0).sum()), "max_ctas_per_sm": int(cnt.max()),
                                            "cluster0_sms": sm[:8].tolist()}
        res[f"{name}_{mode}"] = {f"slot{j}": {"median": float(np.median(rel[:, j])), "max": float(rel[:, j].max()),
                                              "min": float(rel[:, j].min())} for j in range(nslot)}
print(json.dumps(res, indent=1))
