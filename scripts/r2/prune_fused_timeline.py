"""Per-CTA timeline of the fused prune kernel (TL build): TL slots 0 entry,
7 x loaded + squared, 8 cluster wait, 9 pushed, 10 cluster barrier, 11 scores,
13 ranks stored, 12 ranked (flags barrier), 1 ranks/ballots, 2 gathers issued, 3 gathers landed, 4 end."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("RAGGED_LIB", os.path.join(ROOT, "paper_2604_15408_b200", "libragged_tl.so"))
import numpy as np
import torch
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda")
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
lib = rb.lib()
lib.ragged_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
res = {}
for B, H in ((128, 3), (32, 12)):
    N = 197
    kk = synth.kept_tokens(N, 0.8)
    xs = [synth.hidden_states(B, N, H * 64, "bf16", seed=70 + i).to(dev) for i in range(4)]
    q, k, v = (t.to(dev) for t in synth.activations(B, N, H, 64, "bf16", seed=80))
    o = torch.empty_like(q)
    for mode in ("isolated", "back_to_back"):
        for i in range(8):
            rb.prune_l2_pack_attend_unpack(xs[i % 4], q, k, v, kk, o=o)
        torch.cuda.synchronize()
        lib.ragged_debug_timeline_clear()
        if mode == "isolated":
            rb.prune_l2_pack_attend_unpack(xs[1], q, k, v, kk, o=o)
        else:
            for i in range(8):
                rb.prune_l2_pack_attend_unpack(xs[i % 4], q, k, v, kk, o=o)
        torch.cuda.synchronize()
        n = B * H
        buf = np.zeros((n, 16), np.uint64)
        lib.ragged_debug_timeline(buf.ctypes.data, n)
        t = buf[:, :15].astype(np.int64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        d = {}
        for sl in (0, 7, 8, 9, 10, 11, 13, 12, 1, 2, 3, 4):
            d[f"s{sl}"] = [round(float(np.median(rel[:, sl])), 2), round(float(rel[:, sl].max()), 2)]
        d["distinct_sms"] = int(len(set(buf[:, 15].tolist())))
        res[f"B{B}_H{H}_{mode}"] = d
print(json.dumps(res, indent=1))
