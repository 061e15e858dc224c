# speculative prefetch in the packed ragged_attn path: A/B (nopf = none) with scripts/time_separate.py; parity.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
  RAGGED_LIB=paper_2604_15408_b200/libragged_nopf.so timeout 300 python scripts/time_separate.py --config C3 2>/dev/null | tail -1 | sed 's/^/none /' | cut -c1-400
  timeout 300 python scripts/time_separate.py --config C3 2>/dev/null | tail -1 | sed 's/^/spec /' | cut -c1-400
done
timeout 300 python bench.py --no-extras --gather-variants none --cpu-seconds 0.5 --e2e-steps 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('fused C3', round(d['ms_per_step']*1e3,3))"
