"""Per-CTA phase timeline of the fused kernel (needs libragged_tl.so).

    RAGGED_LIB=paper_2604_15408_b200/libragged_tl.so python scripts/timeline.py --config C3
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RAGGED_LIB", os.path.join(ROOT, "paper_2604_15408_b200", "libragged_tl.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_15408_b200 as rb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--prune", type=float, default=None)
ap.add_argument("--engine", type=int, default=0)
ap.add_argument("--out", default="gpurun_out/timeline.json")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
p = c["p"] if a.prune is None else a.prune
H = synth.PRESETS[c["preset"]]["H"]
B, N = c["B"], 197
q, k, v, keep = synth.make_inputs(B, N, H, p, c["method"], "bf16", seed=0)
dev = torch.device("cuda")
S = 16
sets = [[t.to(dev) for t in (q, k, v, keep)] for _ in range(S)]
outs = [torch.empty(B, N, H, 64, dtype=q.dtype, device=dev) for _ in range(S)]
cus = [torch.empty(B + 1, dtype=torch.int32, device=dev) for _ in range(S)]
lib = rb.lib()
lib.ragged_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
lib.ragged_debug_timeline.restype = ctypes.c_int32
ncta = B * H + 1
res = {}
for mode in ("isolated", "back_to_back"):
    for i in range(S):
        rb.pack_attend_unpack(*sets[i], o=outs[i], cu=cus[i], engine=a.engine)
    torch.cuda.synchronize()
    if mode == "isolated":
        rb.pack_attend_unpack(*sets[3], o=outs[3], cu=cus[3], engine=a.engine)
    else:
        for i in range(S):
            rb.pack_attend_unpack(*sets[i], o=outs[i], cu=cus[i], engine=a.engine)
    torch.cuda.synchronize()
    buf = np.zeros((ncta, 16), np.uint64)
    n = lib.ragged_debug_timeline(buf.ctypes.data, ncta)
    assert n == ncta, n
    valid = buf[:, 0] != 0
    t = buf[valid, :13].astype(np.int64)
    sm = buf[valid, 15]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3  # us
    # engine 1: CTA 0 is the scan CTA; engine 2: persistent CTAs (slot 0's last problem)
    attn = rel[1:] if a.engine != 2 else rel
    d = {
        "start_us": np.percentile(attn[:, 0], [0, 50, 90, 100]).tolist(),
        "end_us": np.percentile(attn[:, 4], [0, 50, 90, 100]).tolist(),
        "mask_ballot_us": np.percentile(attn[:, 1] - attn[:, 0], [50, 90, 100]).tolist(),
        "issue_us": np.percentile(attn[:, 2] - attn[:, 1], [50, 90, 100]).tolist(),
        "gather_wait_us": np.percentile(attn[:, 3] - attn[:, 2], [50, 90, 100]).tolist(),
        "compute_store_us": np.percentile(attn[:, 4] - attn[:, 3], [50, 90, 100]).tolist(),
        "w0_qk_softmax_us": np.percentile(attn[:, 5] - attn[:, 3], [50, 90, 100]).tolist(),
        "w0_pv_epi_smem_us": np.percentile(attn[:, 6] - attn[:, 5], [50, 90, 100]).tolist(),
        "w0_store_to_end_us": np.percentile(attn[:, 4] - attn[:, 6], [50, 90, 100]).tolist(),
        "tc_softmax_us": np.percentile(attn[:, 8] - attn[:, 5], [50, 90, 100]).tolist() if a.engine == 2 else None,
        "tc_sm_ld_us": np.percentile(attn[:, 10] - attn[:, 5], [50, 90, 100]).tolist() if a.engine == 2 else None,
        "tc_sm_exp_us": np.percentile(attn[:, 11] - attn[:, 10], [50, 90, 100]).tolist() if a.engine == 2 else None,
        "tc_sm_st_us": np.percentile(attn[:, 12] - attn[:, 11], [50, 90, 100]).tolist() if a.engine == 2 else None,
        "tc_sm_bar_us": np.percentile(attn[:, 8] - attn[:, 12], [50, 90, 100]).tolist() if a.engine == 2 else None,
        "tc_pv_us": np.percentile(attn[:, 9] - attn[:, 8], [50, 90, 100]).tolist() if a.engine == 2 else None,
        "tc_epi_smem_us": np.percentile(attn[:, 6] - attn[:, 9], [50, 90, 100]).tolist() if a.engine == 2 else None,
        "cta_total_us": np.percentile(attn[:, 4] - attn[:, 0], [50, 90, 100]).tolist(),
        "ctas": int(valid.sum()),
        "distinct_sms": int(len(set(sm.tolist()))),
    }
    res[mode] = d
    print(mode, json.dumps(d, indent=1))
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
json.dump({"config": a.config, "p": p, "engine": a.engine, **res}, open(a.out, "w"), indent=1)
