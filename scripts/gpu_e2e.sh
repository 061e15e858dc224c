mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "host" 2>&1 | tail -3
timeout 600 python bench.py --steps 500 --warmup 10 --no-extras --gather-variants none --e2e-steps 100 > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; echo rc=$?
tail -3 gpurun_out/bench_e2e.err
python -c "
import json; d=json.load(open('gpurun_out/bench_e2e.json')); e=d['e2e']
print('us', d['us_per_call']); print(json.dumps(e, indent=1))"
