# Session-3 validation: GPU tests, smoke, full bench (driver args), ncu launch list,
# full capture of the fused C3 kernel and of the WS engine at C3 p=0, cuBLAS kernel names at the block's GEMM shapes.
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/v3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v3_smoke.log 2>&1
timeout 2400 python bench.py --steps 20 --warmup 5 > gpurun_out/v3_bench.json 2> gpurun_out/v3_bench.err
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v3_launches.csv \
  python bench.py --steps 20 --warmup 5 --no-extras --gather-variants none > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_kernel -s 4 -c 2 \
  -o gpurun_out/v3_prof_fused -f python scripts/prof_kernels.py --config C3 --what fused --iters 8 > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_fa -s 2 -c 1 \
  -o gpurun_out/v3_prof_ws_c3p0 -f python scripts/r2/ws_one.py --case c3p0 > /dev/null 2>&1
timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v3_cublas_names.csv \
  python scripts/r2/gemm_split_probe.py > /dev/null 2>&1
echo done > gpurun_out/v3_done.txt
