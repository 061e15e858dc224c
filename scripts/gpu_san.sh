mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 600 $CS --tool $tool --print-limit 20 python scripts/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
timeout 900 python bench.py --steps 2000 --warmup 20 --cpu-seconds 5 --e2e-steps 20 > gpurun_out/bench_full.json 2>gpurun_out/bench_full.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_full.err
