timeout 900 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider -x -k "topk or prune" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; tail -2 gpurun_out/pytest_quick.log
