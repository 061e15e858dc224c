mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1; tail -2 gpurun_out/pytest_quick.log
for e in 1 2; do
  timeout 300 python bench.py --steps 2000 --warmup 20 --engine $e --no-extras --e2e-steps 5 > gpurun_out/bench_e$e.json 2>gpurun_out/bench_e$e.err
  python scripts/timeline.py --config C3 --engine $e --out gpurun_out/tl_c3_e$e.json > /dev/null 2>&1
done
python - <<'PY'
import json
for e in (1,2):
    d=json.load(open(f'gpurun_out/bench_e{e}.json')); print(e, 'us', round(d['us_per_call'],3), 'frac', round(d['roofline']['frac'],3))
    t=json.load(open(f'gpurun_out/tl_c3_e{e}.json'))['back_to_back']
    print({k: [round(x,2) for x in v] if isinstance(v,list) else v for k,v in t.items()})
PY
head -3 gpurun_out/pytest_quick.log 2>/dev/null
