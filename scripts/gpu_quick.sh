mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1; tail -2 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 2000 --warmup 20 --cpu-seconds 2 --e2e-steps 10 > gpurun_out/bench_full.json 2>gpurun_out/bench_full.err; echo bench rc=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_full.json')); x=d['extras']
print('us', round(d['us_per_call'],3), 'frac', round(d['roofline']['frac'],3))
print({k: (round(v,2) if isinstance(v,float) else v) for k,v in x.items() if k not in ('prune_sweep','configs','separate_kernels_roofline')})
print({k: round(v['frac_of_measured_hbm'],3) for k,v in x['separate_kernels_roofline'].items()})
PY
