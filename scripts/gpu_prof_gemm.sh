NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/prof_gemm_qkv -f python scripts/dbg/gemm_one.py 1248 2304 768 0 > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/prof_gemm_fc2 -f python scripts/dbg/gemm_one.py 1248 768 3072 2 > /dev/null 2>&1
echo done
