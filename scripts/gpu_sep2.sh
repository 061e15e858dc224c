mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "scan or pack or composed or unpack or large" 2>&1 | tail -2
for c in "--config C3" "--config C3 --prune 0.0" "--config C4" "--config C1"; do timeout 300 python scripts/time_separate.py $c; done | tee gpurun_out/sep.jsonl
RAGGED_LIB=$PWD/paper_2604_15408_b200/libragged_old.so timeout 300 python scripts/time_separate.py --config C3 | sed "s/^/OLD /"
