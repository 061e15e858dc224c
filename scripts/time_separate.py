"""Device time of the separate path's launches (a1 scan, a2 pack, a3 attn,
a4 unpack, and the 3-call composition) at one config, bench.py protocol
(16 rotating sets, CUDA graphs, cold L2).

    python scripts/time_separate.py --config C3
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_15408_b200 as rb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--prune", type=float, default=None)
ap.add_argument("--reps", type=int, default=500)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
p = c["p"] if a.prune is None else a.prune
H = synth.PRESETS[c["preset"]]["H"]
B, N = c["B"], 197
q, k, v, keep = synth.make_inputs(B, N, H, p, c["method"], "bf16", seed=0)
T = int(keep.numpy().astype(bool).sum())
dev = torch.device("cuda")
S = bench.N_SETS
sets = [dict(q=q.to(dev), k=k.to(dev), v=v.to(dev), keep=keep.to(dev),
             o=torch.empty(B, N, H, 64, dtype=q.dtype, device=dev)) for _ in range(S)]
packed = [rb.pack(s["q"], s["k"], s["v"], s["keep"]) for s in sets]
ops = [torch.empty_like(pk[0]) for pk in packed]
torch.cuda.synchronize()
out = {"config": a.config, "p": p, "T": T}


def sep(i):
    s, pk, o = sets[i], packed[i], ops[i]
    rb.pack(s["q"], s["k"], s["v"], s["keep"], out=pk)
    rb.attn(pk[0], pk[1], pk[2], pk[3], N, op=o)
    rb.unpack(o, pk[4], B, N, o=s["o"])


out["scan_us"] = bench._graph_time(torch, [(lambda i=i: rb.scan(sets[i]["keep"], packed[i][3], packed[i][4],
                                                                packed[i][5])) for i in range(S)], a.reps)
out["pack_us"] = bench._graph_time(torch, [(lambda i=i: rb.pack(sets[i]["q"], sets[i]["k"], sets[i]["v"],
                                                                sets[i]["keep"], out=packed[i]))
                                           for i in range(S)], a.reps)
out["ragged_attn_us"] = bench._graph_time(torch, [(lambda i=i: rb.attn(packed[i][0], packed[i][1], packed[i][2],
                                                                       packed[i][3], N, op=ops[i]))
                                                  for i in range(S)], a.reps)
out["unpack_us"] = bench._graph_time(torch, [(lambda i=i: rb.unpack(ops[i], packed[i][4], B, N, o=sets[i]["o"]))
                                             for i in range(S)], a.reps)
out["separate_path_us"] = bench._graph_time(torch, [(lambda i=i: sep(i)) for i in range(S)], a.reps // 5)
print(json.dumps({k: (round(x, 3) if isinstance(x, float) else x) for k, x in out.items()}), flush=True)
