mkdir -p gpurun_out
timeout 120 python - <<'PY' 2>&1 | tail -8
import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2604_15408_b200 as rb, synth, oracle
for (B,N,H,p,m) in [(1,17,1,0.0,'all'),(2,64,1,0.0,'all'),(4,197,3,0.5,'l2'),(2,197,2,0.0,'all'),(3,197,2,0.8,'l2')]:
    q,k,v,keep = synth.make_inputs(B,N,H,p,m,'bf16',seed=0)
    o = rb.pack_attend_unpack(q.cuda(),k.cuda(),v.cuda(),keep.cuda(), engine=2)
    torch.cuda.synchronize()
    ref,_ = oracle.pack_attend_unpack(q,k,v,keep.numpy())
    err = np.abs(o.double().cpu().numpy()-ref)
    print(B,N,H,p, 'maxerr', err.max(), 'argmax', np.unravel_index(err.argmax(), err.shape))
PY
timeout 900 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1; tail -3 gpurun_out/pytest_quick.log
for e in 1 2; do
  timeout 300 python bench.py --steps 2000 --warmup 20 --engine $e --no-extras --e2e-steps 5 > gpurun_out/bench_e$e.json 2>gpurun_out/bench_e$e.err
  timeout 300 python bench.py --steps 1000 --warmup 20 --engine $e --no-extras --e2e-steps 5 --prune 0.0 > gpurun_out/bench_p0_e$e.json 2>>gpurun_out/bench_e$e.err
done
python - <<'PY'
import json
for e in (1,2):
    for f in (f'gpurun_out/bench_e{e}.json', f'gpurun_out/bench_p0_e{e}.json'):
        try:
            d=json.load(open(f)); print(f, 'us', round(d['us_per_call'],3), 'frac', round(d['roofline']['frac'],3))
        except Exception as ex: print(f, 'ERR', ex)
PY
