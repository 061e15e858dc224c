for v in "" kv64m3 kv64m4 kv64m5; do
  if [ -z "$v" ]; then L=paper_2604_15408_b200/libragged.so; else L=paper_2604_15408_b200/libragged_$v.so; fi
  RAGGED_LIB=$L timeout 300 python scripts/r2/occ_exp.py >> gpurun_out/r2_occ.txt 2>&1
done
