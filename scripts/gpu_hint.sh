# n_hint crossover: headline timing of the short (hint 1) vs long (hint 197) kernel at p in {0.5, 0.6, 0.7, 0.8, 0.9}.
mkdir -p gpurun_out
for p in 0.5 0.6 0.7 0.8 0.9; do for h in 1 197; do
  timeout 300 python bench.py --prune $p --n-hint $h --no-extras --gather-variants none --cpu-seconds 0.5 --e2e-steps 5 > gpurun_out/hint_p${p}_h$h.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/hint_p${p}_h$h.json'));print('p=$p hint=$h', round(d['ms_per_step']*1e3,3),'us')"
done; done
