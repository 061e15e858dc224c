for c in "2 12 0.8 1 host" "3 6 0.5 2 host" "2 12 0.8 1 host_long" "3 6 0.5 2 host_long" "2 12 0.8 1 sleep_default"; do
  timeout 120 python scripts/dbg/gather_cases.py $c 2>&1 | grep CASE
done > gpurun_out/dbg.log
