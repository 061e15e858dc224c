# e2e with the host-link bound (pinned copy-engine bandwidth per direction).
mkdir -p gpurun_out
timeout 600 python bench.py --no-extras --gather-variants none --cpu-seconds 0.5 --e2e-steps 50 > gpurun_out/e2e_bound.json 2>gpurun_out/e2e_bound.err
python -c "import json;d=json.load(open('gpurun_out/e2e_bound.json'));e=d['e2e'];print(e['us_per_step'], e['mode'], e.get('link_bound'))"
