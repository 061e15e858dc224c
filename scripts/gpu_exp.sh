for v in tl tlx; do
RAGGED_LIB=paper_2604_15408_b200/libragged_$v.so python scripts/timeline.py --config C3 --engine 2 --out gpurun_out/${v}_c3_e2.json > /dev/null 2>&1
python -c "
import json
t=json.load(open('gpurun_out/${v}_c3_e2.json'))['back_to_back']; print('$v', {k: [round(x,2) for x in v][:2] if isinstance(v,list) else v for k,v in t.items()})
"
done
for v in "" _x; do RAGGED_LIB=paper_2604_15408_b200/libragged$v.so timeout 300 python bench.py --steps 2000 --warmup 20 --engine 2 --no-extras --e2e-steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lib$v', d['us_per_call'])"; done
