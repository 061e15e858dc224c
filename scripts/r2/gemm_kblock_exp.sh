run() { echo "== $*"; env "$@" timeout 60 python scripts/gemm_probe.py $ARGS; }
for cfg in "128 64 3072 0" "128 256 3072 0" "1248 768 768 0" "1248 768 3072 0"; do
  ARGS=$cfg
  run RAGGED_GEMM_BN=64 RAGGED_GEMM_SPLIT=1
  run RAGGED_GEMM_BN=256 RAGGED_GEMM_SPLIT=1
done
ARGS="1248 768 3072 0"; run RAGGED_GEMM_BN=64 RAGGED_GEMM_SPLIT=1 RAGGED_GEMM_GRID=30
