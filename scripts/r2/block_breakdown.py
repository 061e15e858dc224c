"""N1 block at p = 0.8 (B = 32, T = 1248 live of 6304 capacity rows): every
kernel of ragged_vit_block timed alone (graph replay, weights L2-hot as in the
block bench) beside the torch / cuBLAS op that replaces it."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import bench
import oracle
import paper_2604_15408_b200 as rb
import synth
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
F = torch.nn.functional
dt = torch.bfloat16
pr = synth.PRESETS["deit_base"]
D, H, MLP, N, B = pr["D"], pr["H"], pr["MLP"], 197, 32
res = {}
for p in [float(x) for x in os.environ.get("PROBE_P", "0.8").split(",")]:
    P = {k: v.to(dev) for k, v in synth.vit_weights(D, MLP, dt, 0).items()}
    keep = synth.make_inputs(B, N, H, p, "l2", "bf16", seed=0)[3].numpy()
    cu, _, _ = oracle.scan(keep)
    T = int(cu[-1])
    cud = torch.from_numpy(cu.astype(np.int32)).to(dev)
    live = cud[B:]
    cap = B * N
    x = torch.zeros(cap, D, dtype=dt, device=dev)
    x[:T] = synth.packed_rows(T, D, dt, 0).to(dev)
    y = torch.empty(cap, D, dtype=dt, device=dev)
    qkv = torch.zeros(cap, 3 * D, dtype=dt, device=dev)
    att = torch.zeros(cap, D, dtype=dt, device=dev)
    hmid = torch.zeros(cap, MLP, dtype=dt, device=dev)
    G = lambda f, n=200: bench._graph_time(torch, [f], n)
    q3 = qkv.view(cap, 3, H, 64)
    r = {"T": T}
    r["ln"] = [G(lambda: rb.layer_norm(x, P["ln1_w"], P["ln1_b"], y=y, live=live)),
               G(lambda: F.layer_norm(x[:T], (D,), P["ln1_w"], P["ln1_b"], 1e-6))]
    r["qkv"] = [G(lambda: rb.linear(y, P["w_qkv"], P["b_qkv"], 0, None, out=qkv, live=live)),
                G(lambda: torch.addmm(P["b_qkv"], y[:T], P["w_qkv"].t(), out=qkv[:T]))]
    r["attn"] = [G(lambda: rb.attn(q3[:, 0], q3[:, 1], q3[:, 2], cud, N, op=att.view(cap, H, 64), n_hint=T // B)), None]
    r["proj"] = [G(lambda: rb.linear(att, P["w_proj"], P["b_proj"], 2, x, out=x, live=live)),
                 G(lambda: torch.addmm(x[:T], att[:T], P["w_proj"].t(), out=y[:T]))]
    r["fc1"] = [G(lambda: rb.linear(y, P["w_fc1"], P["b_fc1"], 1, None, out=hmid, live=live)),
                G(lambda: F.gelu(torch.addmm(P["b_fc1"], y[:T], P["w_fc1"].t())))]
    r["fc2"] = [G(lambda: rb.linear(hmid, P["w_fc2"], P["b_fc2"], 2, x, out=x, live=live)),
                G(lambda: torch.addmm(x[:T], hmid[:T], P["w_fc2"].t(), out=y[:T]))]
    blk = rb.VitBlock(P, B, N, H, dt, n_hint=T // B)
    r["block"] = [G(lambda: blk(x, cud), 100), None]
    r["sum_ours"] = sum(v[0] for k, v in r.items() if isinstance(v, list) and k != "block") + r["ln"][0]
    res[f"p{p}"] = r
    print(p, r, flush=True)
print(json.dumps(res))
