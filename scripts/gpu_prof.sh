# ncu evidence for the fused kernel + launch list of a short bench
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_kernel -s 4 -c 2 \
   -o gpurun_out/prof_fused_c3 -f python scripts/prof_kernels.py --config C3 --what fused > gpurun_out/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_kernel -s 4 -c 2 \
   -o gpurun_out/prof_fused_c3p0 -f python scripts/prof_kernels.py --config C3 --prune 0.0 --what fused > gpurun_out/ncu_fused_p0.log 2>&1; echo "ncu fused p0 rc=$?"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 50 --warmup 5 --no-extras --e2e-steps 5 > gpurun_out/launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
   --log-file gpurun_out/launches_sep.csv python scripts/prof_kernels.py --config C3 --what attn,pack,unpack,scan --iters 10 > /dev/null 2>&1; echo "ncu sep rc=$?"
ls -la gpurun_out
