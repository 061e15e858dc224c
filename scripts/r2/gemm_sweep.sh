# BN x split sweep of the four DeiT-B GEMM shapes (env read once per process)
for bn in 64 128 192 256; do for sp in 1 2 4; do
  RAGGED_GEMM_BN=$bn RAGGED_GEMM_SPLIT=$sp PROBE_T=${PROBE_T:-1248,6304} timeout 120 python scripts/r2/gemm_split_probe.py | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bn=$bn sp=$sp', ' '.join(f'{k}={v[\"ours_us\"]:.2f}' for k,v in d.items() if isinstance(v,dict)))"
done; done
