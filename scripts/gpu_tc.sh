mkdir -p gpurun_out
timeout 120 python - <<'PY' 2>&1 | tail -20
import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2604_15408_b200 as rb, synth, oracle
for (B,N,H,p,m) in [(1,17,1,0.0,'all'),(2,64,1,0.0,'all'),(4,197,3,0.5,'l2'),(2,197,2,0.0,'all')]:
    q,k,v,keep = synth.make_inputs(B,N,H,p,m,'bf16',seed=0)
    o = rb.pack_attend_unpack(q.cuda(),k.cuda(),v.cuda(),keep.cuda(), engine=2)
    torch.cuda.synchronize()
    ref,_ = oracle.pack_attend_unpack(q,k,v,keep.numpy())
    err = np.abs(o.double().cpu().numpy()-ref)
    print(B,N,H,p, 'maxerr', err.max(), 'argmax', np.unravel_index(err.argmax(), err.shape))
PY
timeout 600 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider -x 2>&1 | tail -15
