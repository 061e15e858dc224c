# ViT block with n_hint: parity (every hint) and the bench's n1_block extras.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_block.py -m gpu -q -x 2>&1 | tail -1
timeout 900 python - <<'PY'
import json, sys, types
sys.argv = ["bench.py"]
import bench, torch
import paper_2604_15408_b200 as rb
PY
timeout 900 python bench.py --gather-variants none --cpu-seconds 0.5 --e2e-steps 5 > gpurun_out/bh_bench.json 2>gpurun_out/bh_bench.err
python -c "import json;d=json.load(open('gpurun_out/bh_bench.json'));print(json.dumps(d['extras']['n1_block'])[:900])"
