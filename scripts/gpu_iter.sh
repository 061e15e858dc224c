# quick iteration: fused parity tests + C3 / sweep timings of the current build
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gather.py -q -x -p no:cacheprovider 2>&1 | tail -3
for pr in 0.8 0.9 0.7 0.5 0.3 0.0; do
  timeout 120 python scripts/ablate.py --config C3 --prune $pr --tag "cur" 2>&1 | tail -1
done | tee gpurun_out/iter.jsonl
timeout 120 python scripts/ablate.py --config C3 --no-cu --tag "cur nocu" 2>&1 | tail -1
for v in abz abc aball; do
  RAGGED_LIB=$PWD/paper_2604_15408_b200/libragged_$v.so timeout 120 python scripts/ablate.py --config C3 --tag "$v" 2>&1 | tail -1
done
