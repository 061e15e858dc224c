mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_ws.py -x -q > gpurun_out/j7_pytest_ws.log 2>&1
L=$PWD/paper_2604_15408_b200
for v in head poly0 poly1 "" poly3 poly4; do
  if [ -z "$v" ]; then lib=$L/libragged.so; n=poly2; else lib=$L/libragged_$v.so; n=$v; fi
  RAGGED_LIB=$lib timeout 600 python scripts/r2/ws_cross.py > gpurun_out/j7_cross_$n.log 2>&1
done
CASE=c3p0 timeout 120 python scripts/r2/ws_tl2.py > gpurun_out/j7_tl_c3p0.json 2>&1
