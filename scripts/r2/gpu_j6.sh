mkdir -p gpurun_out
for c in c3p05 c3p0 vitl; do CASE=$c timeout 120 python scripts/r2/ws_tl2.py > gpurun_out/j6_tl_$c.json 2>&1; done
