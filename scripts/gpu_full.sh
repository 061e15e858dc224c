NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_kernel -s 4 -c 2 \
   -o gpurun_out/prof_traffic -f python scripts/prof_kernels.py --config C3 --what fused --iters 8 > /dev/null 2>&1; echo ncu rc=$? > gpurun_out/ncu_rc.txt
timeout 1500 python bench.py --steps 2000 --warmup 20 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
