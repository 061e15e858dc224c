# Long-sequence chunk experiment: parity of the n_hint kernel, then the headline at p in {0, .3, .5, .7, .8}.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "long_sequence or fused_baseline or c5_scale" > gpurun_out/lazy_pytest.log 2>&1; tail -2 gpurun_out/lazy_pytest.log
for p in 0.0 0.3 0.5 0.7 0.8; do
  timeout 300 python bench.py --prune $p --no-extras --gather-variants none --cpu-seconds 0.5 --e2e-steps 5 > gpurun_out/lazy_p$p.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/lazy_p$p.json'));print('p=$p', round(d['ms_per_step']*1e3,3),'us')"
done
