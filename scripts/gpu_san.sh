mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python scripts/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?" >> gpurun_out/sanitize_rc.txt
done
