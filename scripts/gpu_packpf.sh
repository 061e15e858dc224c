# pre-wait prefetch in the small-batch scan/pack kernel: A/B (nopf) via scripts/time_separate.py; GPU suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
  RAGGED_LIB=paper_2604_15408_b200/libragged_nopf.so timeout 300 python scripts/time_separate.py --config C3 2>/dev/null | tail -1 | sed 's/^/none /' | cut -c1-300
  timeout 300 python scripts/time_separate.py --config C3 2>/dev/null | tail -1 | sed 's/^/with /' | cut -c1-300
done
