mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for e in 1 2; do
  K=attn_kernel; [ $e = 2 ] && K=attn_tc_kernel
  timeout 600 $NCU --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:$K -s 6 -c 1 \
     -o gpurun_out/prof_e${e}_c3 -f python scripts/prof_kernels.py --config C3 --what fused --engine $e --iters 10 > gpurun_out/ncu_e$e.log 2>&1; echo "ncu e$e rc=$?"
done
