mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gather.py -q -x -p no:cacheprovider 2>&1 | tail -2
for cfg in "--config C3" "--config C4" "--config C5 --steps 50 --sets 2"; do
  timeout 200 python scripts/ablate.py $cfg --tag "cu" 2>&1 | tail -1 | sed 's/"all.*//'
  timeout 200 python scripts/ablate.py $cfg --tag "nocu" --no-cu 2>&1 | tail -1 | sed 's/"all.*//'
done | tee gpurun_out/cu.jsonl
