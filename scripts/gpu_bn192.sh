# GEMM tile width 192: parity with the cost model's choice and with BN forced to 192; timings per forced BN.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_block.py -m gpu -q -x 2>&1 | tail -1
RAGGED_GEMM_BN=192 timeout 600 python -m pytest tests/test_gpu_block.py -m gpu -q -x 2>&1 | tail -1
for bn in auto 128 192 256; do
  if [ $bn = auto ]; then unset RAGGED_GEMM_BN; else export RAGGED_GEMM_BN=$bn; fi
  timeout 600 python scripts/bench_block.py 1248 6304 50000 > gpurun_out/bn_$bn.json 2>/dev/null
  python - $bn <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/bn_{sys.argv[1]}.json"))
print(sys.argv[1], {T:{k:round(v['ours_us'],1) for k,v in r.items() if isinstance(v,dict)} for T,r in d.items() if T.startswith('T=')},
      {k:round(v['ours_us'],1) for k,v in d.items() if k.startswith('block')})
PY
done
unset RAGGED_GEMM_BN
