mkdir -p gpurun_out
for e in 1 2; do
  python scripts/timeline.py --config C3 --engine $e --out gpurun_out/tl_c3_e$e.json > /dev/null 2>&1
  python scripts/timeline.py --config C3 --prune 0.0 --engine $e --out gpurun_out/tl_c3p0_e$e.json > /dev/null 2>&1
  timeout 300 python bench.py --steps 2000 --warmup 20 --engine $e --cpu-seconds 2 --e2e-steps 5 > gpurun_out/bench_e$e.json 2>gpurun_out/bench_e$e.err
done
python - <<'PY'
import json
for e in (1,2):
    d=json.load(open(f'gpurun_out/bench_e{e}.json'))
    x=d.get('extras',{})
    print('engine',e,'fused us',round(d['us_per_call'],3),'frac',round(d['roofline']['frac'],3),'attn us',round(x.get('ragged_attn_us',0),3))
    print('  sweep', [(s['p'], round(s['fused_us'],2)) for s in x.get('prune_sweep',[])])
    for f in (f'gpurun_out/tl_c3_e{e}.json', f'gpurun_out/tl_c3p0_e{e}.json'):
        t=json.load(open(f))['back_to_back']
        print('  ', f.split('/')[-1], {k: [round(v,2) for v in vv] if isinstance(vv,list) else vv for k,vv in t.items()})
PY
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 4 -c 2 -o gpurun_out/prof_tc_c3 -f python scripts/prof_kernels.py --config C3 --what fused --engine 2 > /dev/null 2>&1; echo ncu1 $?
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 4 -c 2 -o gpurun_out/prof_tc_c3p0 -f python scripts/prof_kernels.py --config C3 --prune 0.0 --what fused --engine 2 > /dev/null 2>&1; echo ncu2 $?
