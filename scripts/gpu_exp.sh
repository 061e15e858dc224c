python scripts/timeline.py --config C3 --engine 2 --prune 0.0 --out gpurun_out/tl_p0_e2.json > /dev/null 2>&1
python -c "
import json
d=json.load(open('gpurun_out/tl_p0_e2.json'))
for m in ('isolated','back_to_back'):
  t=d[m]; print(m, {k: [round(x,2) for x in v] if isinstance(v,list) else v for k,v in t.items() if v is not None and 'sm_' not in k})
"
