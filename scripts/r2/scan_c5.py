"""Separate path pieces at C5 (DeiT-B, B = 4096, 70 %): ragged_scan / ragged_pack / ragged_attn /
ragged_unpack vs the fused call (graph replay)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
B, N, H, p = 4096, 197, 12, 0.7
q, k, v, keep = (t.to(dev) for t in synth.make_inputs(B, N, H, p, "l2", "bf16", seed=0))
kk = synth.kept_tokens(N, p)
cu = torch.empty(B + 1, dtype=torch.int32, device=dev)
dst = torch.empty(B * N, dtype=torch.int32, device=dev)
src = torch.empty(B * N, dtype=torch.int32, device=dev)
qp, kp, vp, cu2, dst2, src2 = rb.pack(q, k, v, keep)
op = torch.empty_like(qp)
o = torch.empty(B, N, H, 64, dtype=torch.bfloat16, device=dev)
torch.cuda.synchronize()
res = {"scan_us": bench._graph_time(torch, [lambda: rb.scan(keep, cu, dst, src)], 20),
       "pack_us": bench._graph_time(torch, [lambda: rb.pack(q, k, v, keep, out=(qp, kp, vp, cu2, dst2, src2))], 10),
       "attn_us": bench._graph_time(torch, [lambda: rb.attn(qp, kp, vp, cu2, N, op=op, n_hint=kk)], 10),
       "unpack_us": bench._graph_time(torch, [lambda: rb.unpack(op, dst2, B, N, o=o)], 10),
       "fused_us": bench._graph_time(torch, [lambda: rb.pack_attend_unpack(q, k, v, keep, o=o, cu=cu, n_hint=kk)], 10)}
print(json.dumps(res))
