NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:attn_kernel -s 6 -c 1 \
   -o gpurun_out/prof_mma_p0 -f python scripts/prof_kernels.py --config C3 --prune 0.0 --what fused --engine 1 --iters 10 > /dev/null 2>&1; echo ncu rc=$?
