mkdir -p gpurun_out
python scripts/timeline.py --config C3 --out gpurun_out/tl_c3.json 2>&1 | tail -60
timeout 300 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider 2>&1 | tail -3
timeout 300 python bench.py --steps 2000 --warmup 20 --no-extras --e2e-steps 5 > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err; python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json')); print('us_per_call', d['us_per_call'], 'frac', d['roofline']['frac'], d['clocks'])"
