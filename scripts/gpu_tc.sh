mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider -x 2>&1 | tail -6
for e in 2; do
  python scripts/timeline.py --config C3 --engine $e --out gpurun_out/tl_c3_e$e.json > /dev/null 2>&1
  python scripts/timeline.py --config C3 --prune 0.0 --engine $e --out gpurun_out/tl_c3p0_e$e.json > /dev/null 2>&1
done
for e in 1 2; do
  timeout 300 python bench.py --steps 2000 --warmup 20 --engine $e --no-extras --e2e-steps 5 > gpurun_out/bench_e$e.json 2>gpurun_out/bench_e$e.err
  timeout 300 python bench.py --steps 1000 --warmup 20 --engine $e --no-extras --e2e-steps 5 --prune 0.0 > gpurun_out/bench_p0_e$e.json 2>>gpurun_out/bench_e$e.err
  timeout 300 python bench.py --steps 200 --warmup 5 --engine $e --no-extras --e2e-steps 2 --config C5 > gpurun_out/bench_c5_e$e.json 2>>gpurun_out/bench_e$e.err
done
python - <<'PY'
import json
for e in (1,2):
    for f in (f'gpurun_out/bench_e{e}.json', f'gpurun_out/bench_p0_e{e}.json', f'gpurun_out/bench_c5_e{e}.json'):
        try:
            d=json.load(open(f)); print(f, 'us', round(d['us_per_call'],3), 'frac', round(d['roofline']['frac'],3))
        except Exception as ex: print(f, 'ERR', ex)
for f in ('gpurun_out/tl_c3_e2.json','gpurun_out/tl_c3p0_e2.json'):
    t=json.load(open(f))['back_to_back']
    print(f, {k: [round(x,2) for x in v] if isinstance(v,list) else v for k,v in t.items()})
PY
tail -3 gpurun_out/bench_e2.err
