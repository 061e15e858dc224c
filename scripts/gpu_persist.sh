mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for cfg in "--config C3" "--config C3 --prune 0.0" "--config C4" "--config C4 --prune 0.9" "--config C5 --steps 50 --sets 2"; do
  for ps in 1 0; do RAGGED_PERSIST=$ps timeout 200 python scripts/ablate.py $cfg --tag "persist=$ps" 2>&1 | tail -1 | sed 's/"all.*//'; done
done | tee gpurun_out/persist.jsonl
