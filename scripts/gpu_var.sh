# timings of experiment builds: bash scripts/gpu_var.sh "zb za" "0.8 0.5 0.0"
mkdir -p gpurun_out
for pr in $2; do
for v in "" $1; do
  lib=paper_2604_15408_b200/libragged${v:+_$v}.so
  RAGGED_LIB=$PWD/$lib timeout 120 python scripts/ablate.py --config C3 --prune $pr --tag "$v" 2>&1 | tail -1
done
done | tee gpurun_out/var.jsonl
