mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/j1_smi.txt
timeout 600 python scripts/r2/ws_quick.py > gpurun_out/j1_ws_quick.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/j1_bench.json 2> gpurun_out/j1_bench.err
