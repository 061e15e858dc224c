mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ws.py tests/test_gpu_block.py tests/test_gpu_pipeline.py -x -q > gpurun_out/j8_pytest.log 2>&1
PROBE_P=0.8,0.0 timeout 300 python scripts/r2/block_breakdown.py > gpurun_out/j8_block.log 2>&1
timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/j8_gemm_default.json 2>&1
RAGGED_GEMM_SPLIT=1 timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/j8_gemm_split1.json 2>&1
RAGGED_GEMM_SPLIT=1 RAGGED_GEMM_BN=64 timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/j8_gemm_bn64.json 2>&1
RAGGED_GEMM_SPLIT=1 RAGGED_GEMM_BN=128 timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/j8_gemm_bn128.json 2>&1
RAGGED_GEMM_SPLIT=2 RAGGED_GEMM_BN=64 timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/j8_gemm_s2bn64.json 2>&1
timeout 200 python scripts/r2/prune_timeline.py > gpurun_out/j8_prune_tl.json 2>&1
