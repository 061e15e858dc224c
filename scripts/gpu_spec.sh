# speculative kept-row prefetch (libragged_spec.so) vs keep-row prefetch (default) vs none (nopf).
mkdir -p gpurun_out
RAGGED_LIB=paper_2604_15408_b200/libragged_spec.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused or host or graph" 2>&1 | tail -1
run() { timeout 300 python bench.py $1 --no-extras --gather-variants none --cpu-seconds 0.5 --e2e-steps 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$2', '$1', round(d['ms_per_step']*1e3,3),'us', 'e2e', round(d['e2e']['us_per_step'],1))"; }
for args in "--prune 0.8" "--prune 0.9" "--prune 0.5" "--prune 0.0" "--config C4" "--config C5 --steps 200"; do
  for r in 1 2; do
    RAGGED_LIB=paper_2604_15408_b200/libragged_nopf.so run "$args" none
    run "$args" keep
    RAGGED_LIB=paper_2604_15408_b200/libragged_spec.so run "$args" spec
  done
done
