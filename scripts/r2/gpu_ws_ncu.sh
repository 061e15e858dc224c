mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_fa -s 2 -c 1 -o gpurun_out/r2_ws_vitl -f python scripts/r2/ws_one.py --case vitl > gpurun_out/r2_ws_ncu.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_fa -s 2 -c 1 -o gpurun_out/r2_ws_c3p0 -f python scripts/r2/ws_one.py --case c3p0 >> gpurun_out/r2_ws_ncu.log 2>&1
