# e2e with host-resident O zeroed early (during the gathers); host-input parity tests; device headline unchanged.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host or fused_baseline" > gpurun_out/ze_pytest.log 2>&1; tail -2 gpurun_out/ze_pytest.log
timeout 600 python bench.py --no-extras --gather-variants none --cpu-seconds 0.5 --e2e-steps 50 > gpurun_out/ze_bench.json 2>gpurun_out/ze_bench.err
python - <<'PY'
import json;d=json.load(open('gpurun_out/ze_bench.json'));e=d['e2e']
print('device us', round(d['ms_per_step']*1e3,3))
for k,v in e['variants'].items(): print(k, round(v.get('us_per_step',0),1))
print(e.get('link_bound'))
PY
