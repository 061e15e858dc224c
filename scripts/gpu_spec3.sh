# verified speculative ranks: full GPU suite, then headline at p in {0.8, 0.9, 0.5, 0.0}, C4, C5.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
run() { timeout 300 python bench.py $1 --no-extras --gather-variants none --cpu-seconds 0.5 --e2e-steps 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$1', round(d['ms_per_step']*1e3,3),'us')"; }
for args in "--prune 0.8" "--prune 0.8" "--prune 0.9" "--prune 0.5" "--prune 0.0" "--config C4" "--config C5 --steps 200"; do run "$args"; done
