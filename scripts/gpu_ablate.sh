# Ablation timings of the fused kernel (C3 and p=0): full / no zero rows / no compute / neither
mkdir -p gpurun_out
for cfg in "--config C3" "--config C3 --prune 0.5"; do
for v in "" abz abc aball; do
  lib=paper_2604_15408_b200/libragged${v:+_$v}.so
  RAGGED_LIB=$PWD/$lib timeout 120 python scripts/ablate.py $cfg --tag "$v" 2>&1 | tail -1
  RAGGED_LIB=$PWD/$lib timeout 120 python scripts/ablate.py $cfg --tag "$v nocu" --no-cu 2>&1 | tail -1
done
done | tee gpurun_out/ablate.jsonl
