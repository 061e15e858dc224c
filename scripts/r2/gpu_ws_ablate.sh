for v in "" fansm fanpv fanone; do
  if [ -z "$v" ]; then L=paper_2604_15408_b200/libragged.so; else L=paper_2604_15408_b200/libragged_$v.so; fi
  RAGGED_LIB=$L timeout 300 python scripts/r2/ws_ablate.py >> gpurun_out/r2_ws_ablate.txt 2>&1
done
