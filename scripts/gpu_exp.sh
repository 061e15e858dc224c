python scripts/timeline.py --config C3 --engine 2 --out gpurun_out/tl_c3_e2.json > /dev/null 2>&1
python -c "
import json
t=json.load(open('gpurun_out/tl_c3_e2.json'))['back_to_back']; print({k: [round(x,2) for x in v] if isinstance(v,list) else v for k,v in t.items() if k.startswith('tc')})
"
