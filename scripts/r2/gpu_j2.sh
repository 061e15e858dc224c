mkdir -p gpurun_out
timeout 300 python scripts/r2/headline_fixed.py > gpurun_out/j2_fixed.log 2>&1
timeout 600 python scripts/r2/ws_cross.py > gpurun_out/j2_cross_base.log 2>&1
RAGGED_LIB=$PWD/paper_2604_15408_b200/libragged_fap16.so timeout 600 python scripts/r2/ws_cross.py > gpurun_out/j2_cross_p16.log 2>&1
