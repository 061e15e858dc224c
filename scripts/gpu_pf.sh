# keep-row L2 prefetch before the PDL wait: A/B (libragged_nopf.so = without) at p in {0.9, 0.8, 0.7}, C1, C4, C5.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused or host or graph" 2>&1 | tail -1
run() { timeout 300 python bench.py $1 --no-extras --gather-variants none --cpu-seconds 0.5 --e2e-steps 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$2', '$1', round(d['ms_per_step']*1e3,3),'us')"; }
for args in "--prune 0.9" "--prune 0.8" "--prune 0.7" "--config C1" "--config C4" "--config C5 --steps 200"; do
  for r in 1 2; do
    RAGGED_LIB=paper_2604_15408_b200/libragged_nopf.so run "$args" without
    run "$args" with
  done
done
