# Validation recipe (run on the GPU box from the repo root, e.g.
#   gpurun --timeout 3600 -- 'bash scripts/gpu_validate.sh'):
# GPU tests, smoke, the bench line with the driver's arguments, the ncu launch
# list of the same command, full ncu captures of the fused C3 kernel and of the
# warp-specialised engine at C3 p = 0, the window DRAM traffic of the fused
# kernel (roofline.traffic), and cuBLAS's kernels at the N1 block's GEMM shapes.
# Outputs land in gpurun_out/val_*; summaries worth keeping go to profiles/.
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/val_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1
timeout 2400 python bench.py --steps 20 --warmup 5 > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/val_launches.csv \
  python bench.py --steps 20 --warmup 5 --no-extras --gather-variants none > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_kernel -s 4 -c 2 \
  -o gpurun_out/val_prof_fused -f python scripts/prof_kernels.py --config C3 --what fused --iters 8 > /dev/null 2>&1
timeout 600 $NCU --replay-mode range --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/val_traffic_range.csv python scripts/r2/traffic_range.py > gpurun_out/val_traffic_range.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_fa -s 2 -c 1 \
  -o gpurun_out/val_prof_ws_c3p0 -f python scripts/r2/ws_one.py --case c3p0 > /dev/null 2>&1
timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/val_cublas_names.csv \
  python scripts/r2/gemm_split_probe.py > /dev/null 2>&1
echo done > gpurun_out/val_done.txt
