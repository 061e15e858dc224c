import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import oracle, synth
import paper_2604_15408_b200 as rb
import test_gpu_block as t
for preset, B, p, method in [("deit_tiny", 4, 0.5, "l2"), ("deit_small", 6, 0.0, "l2"), ("deit_base", 8, 0.8, "l2"),
                             ("deit_base", 5, 0.7, "ats"), ("deit_base", 8, 0.0, "l2"), ("deit_base", 32, 0.8, "l2")]:
    params, cu, x, D, H, MLP, N, T = t._block_inputs(preset, B, p, seed=B, method=method)
    blk = rb.VitBlock({k: v.to("cuda") for k, v in params.items()}, B, N, H, torch.bfloat16)
    xd = torch.zeros(B * N, D, dtype=torch.bfloat16, device="cuda"); xd[:T] = x.cuda()
    blk(xd, torch.from_numpy(cu.astype(np.int32)).cuda()); torch.cuda.synchronize()
    got = xd[:T].double().cpu().numpy()
    ref = oracle.vit_block(x, cu, params, H, store=t.store(torch.bfloat16))
    ref64 = oracle.vit_block(x, cu, params, H)
    err = np.abs(got - ref); u = t.ulp(ref, torch.bfloat16)
    e64 = np.abs(got - ref64); e_st = np.abs(ref - ref64)
    print(preset, B, p, method, "T", T, "max|ref| %.3f" % np.abs(ref).max(),
          "maxerr %.4f (%.5f of max)" % (err.max(), err.max() / np.abs(ref).max()),
          "relF %.2e" % (np.linalg.norm(got - ref) / np.linalg.norm(ref)),
          "<=1ulp %.5f <=2ulp %.5f <=4ulp %.6f" % ((err <= u).mean(), (err <= 2 * u).mean(), (err <= 4 * u).mean()),
          "| vs fp64: gpu relF %.2e  oracle-stored relF %.2e" % (np.linalg.norm(got - ref64) / np.linalg.norm(ref64),
                                                                  np.linalg.norm(ref - ref64) / np.linalg.norm(ref64)))
