mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_pipeline.py -q -rf --tb=short -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/t4_pytest.log
timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/t4_gemm_default.json 2>&1
RAGGED_GEMM_MCAST=1 timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/t4_gemm_mc1.json 2>&1
RAGGED_GEMM_SPLIT=1 timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/t4_gemm_s1mc.json 2>&1
RAGGED_GEMM_SPLIT=1 RAGGED_GEMM_MCAST=2 timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/t4_gemm_s1mc2.json 2>&1
RAGGED_GEMM_SPLIT=1 RAGGED_GEMM_BN=128 timeout 200 python scripts/r2/gemm_split_probe.py > gpurun_out/t4_gemm_s1bn128mc.json 2>&1
PROBE_P=0.8,0.0 timeout 300 python scripts/r2/block_breakdown.py > gpurun_out/t4_block.log 2>&1
RAGGED_GEMM_SPLIT=1 PROBE_P=0.8,0.0 timeout 300 python scripts/r2/block_breakdown.py > gpurun_out/t4_block_s1.log 2>&1
