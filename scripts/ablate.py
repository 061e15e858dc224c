"""Device time of the fused call at one config for one build of the library
(timing experiments; select the build with RAGGED_LIB).  Same protocol as
bench.py: 16 rotating input/output sets (> L2), K calls in one CUDA graph.

    RAGGED_LIB=paper_2604_15408_b200/libragged_abz.so python scripts/ablate.py --config C3
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_15408_b200 as rb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--prune", type=float, default=None)
ap.add_argument("--engine", type=int, default=0)
ap.add_argument("--steps", type=int, default=1000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-cu", action="store_true")
ap.add_argument("--tag", default="")
ap.add_argument("--sets", type=int, default=16)
ap.add_argument("--n-hint", type=int, default=0)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
p = c["p"] if a.prune is None else a.prune
H = synth.PRESETS[c["preset"]]["H"]
B, N = c["B"], 197
q, k, v, keep = synth.make_inputs(B, N, H, p, c["method"], "bf16", seed=0)
dev = torch.device("cuda")
S = a.sets
sets = [[t.to(dev) for t in (q, k, v, keep)] for _ in range(S)]
outs = [torch.empty(B, N, H, 64, dtype=q.dtype, device=dev) for _ in range(S)]
cus = [torch.empty(B + 1, dtype=torch.int32, device=dev) for _ in range(S)]
for i in range(20):
    rb.pack_attend_unpack(*sets[i % S], o=outs[i % S], cu=None if a.no_cu else cus[i % S], engine=a.engine,
                          n_hint=a.n_hint)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream()
with torch.cuda.graph(g, stream=cap):
    for i in range(a.steps):
        rb.pack_attend_unpack(*sets[i % S], o=outs[i % S], cu=None if a.no_cu else cus[i % S],
                              engine=a.engine, n_hint=a.n_hint)
g.replay()
torch.cuda.synchronize()
us = []
for _ in range(a.reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    us.append(1e3 * s.elapsed_time(e) / a.steps)
print(json.dumps({"lib": os.path.basename(rb.LIB_PATH), "tag": a.tag, "config": a.config, "p": p,
                  "engine": a.engine, "us": sorted(us)[len(us) // 2], "all": us}), flush=True)
