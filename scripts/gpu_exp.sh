mkdir -p gpurun_out
for v in tl tlx; do
RAGGED_LIB=paper_2604_15408_b200/libragged_$v.so python scripts/timeline.py --config C3 --engine 2 --out gpurun_out/${v}_c3_e2.json > /dev/null 2>&1
python -c "
import json
d=json.load(open('gpurun_out/${v}_c3_e2.json'))
t=d['back_to_back']; print('$v', {k: [round(x,2) for x in v] if isinstance(v,list) else v for k,v in t.items()})
"
done
