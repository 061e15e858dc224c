python scripts/timeline.py --config C3 --engine 2 --prune 0.0 --out gpurun_out/tl_p0_e2.json > /dev/null 2>&1
python scripts/timeline.py --config C3 --engine 2 --out gpurun_out/tl_c3_e2.json > /dev/null 2>&1
for f in tl_p0_e2 tl_c3_e2; do python -c "
import json
t=json.load(open('gpurun_out/$f.json'))['back_to_back']; print('$f', {k: [round(x,2) for x in v][:2] if isinstance(v,list) else v for k,v in t.items()})
"; done
