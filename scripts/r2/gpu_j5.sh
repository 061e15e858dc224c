mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
RAGGED_LIB=$PWD/paper_2604_15408_b200/libragged_head.so timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_fa -s 2 -c 1 -o gpurun_out/j5_ws_c3p05 -f python scripts/r2/ws_one.py --case c3p05 > gpurun_out/j5_ncu.log 2>&1
RAGGED_LIB=$PWD/paper_2604_15408_b200/libragged_head.so timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_fa -s 2 -c 1 -o gpurun_out/j5_ws_c3p0 -f python scripts/r2/ws_one.py --case c3p0 >> gpurun_out/j5_ncu.log 2>&1
