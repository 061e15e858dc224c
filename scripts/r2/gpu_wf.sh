mkdir -p gpurun_out
timeout 600 python scripts/r2/ws_fused_check.py > gpurun_out/wf.log 2>&1
