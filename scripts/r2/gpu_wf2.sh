mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ws.py -q -rf --tb=short -p no:cacheprovider 2>&1 | tail -6 > gpurun_out/wf2_pytest.log
timeout 600 python scripts/r2/ws_fused_check.py > gpurun_out/wf2.log 2>&1
FUSED=1 CASE=c3p0 timeout 120 python scripts/r2/ws_tl2.py > gpurun_out/wtl2_fused.json 2>&1
