mkdir -p gpurun_out
python scripts/timeline.py --config C3 --out gpurun_out/tl_c3.json 2>&1 | tail -40
python scripts/timeline.py --config C3 --prune 0.0 --out gpurun_out/tl_c3p0.json 2>&1 | tail -40
