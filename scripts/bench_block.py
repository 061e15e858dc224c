"""N1 microbench: tcgen05 GEMM vs cuBLAS (torch.nn.functional.linear) on the
block's shapes, LayerNorm, and the whole packed block; device time from CUDA
graphs of `reps` calls."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2604_15408_b200 as rb
import synth, oracle

def gtime(fn, reps=200):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps): fn()
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / reps

out = {}
D, H, MLP = 768, 12, 3072
dt = torch.bfloat16
for T in [int(a) for a in (sys.argv[1:] or ["1248", "6304", "50000"])]:
    res = {}
    for name, N, K, epi in [("qkv", 3 * D, D, 0), ("proj", D, D, 2), ("fc1", MLP, D, 1), ("fc2", D, MLP, 2)]:
        a = torch.randn(T, K, device="cuda").to(dt)
        w = (0.02 * torch.randn(N, K, device="cuda")).to(dt)
        bias = torch.zeros(N, device="cuda", dtype=dt)
        r = torch.randn(T, N, device="cuda").to(dt)
        o = torch.empty(T, N, device="cuda", dtype=dt)
        ours = gtime(lambda: rb.linear(a, w, bias, epi, r if epi == 2 else None, out=o))
        if epi == 1:
            ref = lambda: torch.nn.functional.gelu(torch.nn.functional.linear(a, w, bias))
        elif epi == 2:
            ref = lambda: torch.add(torch.nn.functional.linear(a, w, bias), r)
        else:
            ref = lambda: torch.nn.functional.linear(a, w, bias)
        cub = gtime(ref)
        plain = gtime(lambda: torch.nn.functional.linear(a, w))
        fl = 2.0 * T * N * K
        res[name] = {"ours_us": ours, "torch_fused_equiv_us": cub, "cublas_gemm_only_us": plain,
                     "ours_tflops": fl / ours / 1e6, "cublas_tflops": fl / plain / 1e6}
    x = torch.randn(T, D, device="cuda").to(dt); w1 = torch.ones(D, device="cuda", dtype=dt); b1 = torch.zeros_like(w1)
    y = torch.empty_like(x)
    res["layer_norm_us"] = gtime(lambda: rb.layer_norm(x, w1, b1, y=y))
    res["torch_layer_norm_us"] = gtime(lambda: torch.nn.functional.layer_norm(x, (D,), w1, b1, 1e-6))
    out[f"T={T}"] = res

# whole block, DeiT-B, B=32, p in {0.8, 0.0}: ours vs a torch packed block (cuBLAS linears + our attention)
for p in (0.8, 0.0):
    B, N = 32, 197
    params = {k: v.cuda() for k, v in synth.vit_weights(D, MLP, dt, 0).items()}
    keep = synth.make_inputs(B, N, H, p, "l2", "bf16", seed=0)[3].numpy()
    cu, _, _ = oracle.scan(keep); T = int(cu[-1])
    cud = torch.from_numpy(cu.astype(np.int32)).cuda()
    blk = rb.VitBlock(params, B, N, H, dt)
    x = torch.zeros(B * N, D, device="cuda", dtype=dt); x[:T] = synth.packed_rows(T, D, dt, 0).cuda()
    ours = gtime(lambda: blk(x, cud), reps=100)
    P = params
    def torch_block(xx=x[:T]):
        y = torch.nn.functional.layer_norm(xx, (D,), P["ln1_w"], P["ln1_b"], 1e-6)
        qkv = torch.nn.functional.linear(y, P["w_qkv"], P["b_qkv"]).view(T, 3, H, 64)
        a = rb.attn(qkv[:, 0], qkv[:, 1], qkv[:, 2], cud, N)
        h = xx + torch.nn.functional.linear(a.view(T, D), P["w_proj"], P["b_proj"])
        z = torch.nn.functional.layer_norm(h, (D,), P["ln2_w"], P["ln2_b"], 1e-6)
        f = torch.nn.functional.gelu(torch.nn.functional.linear(z, P["w_fc1"], P["b_fc1"]))
        return h + torch.nn.functional.linear(f, P["w_fc2"], P["b_fc2"])
    tb = gtime(torch_block, reps=100)
    fl = 2.0 * T * D * (3 * D + D + 2 * MLP) + 4.0 * float((np.diff(cu) ** 2).sum()) * 64 * H
    out[f"block_B32_p{p}"] = {"T": T, "ours_us": ours, "torch_cublas_plus_our_attn_us": tb,
                              "ours_tflops": fl / ours / 1e6, "images_per_s": B / ours * 1e6}
print(json.dumps(out, indent=1))
