mkdir -p gpurun_out/s19
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s19/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s19/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/s19/bench.json 2> gpurun_out/s19/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/s19/bench.json').read().strip().splitlines()[-1])
print('headline', d['value'], d['ms_per_step'], d['roofline']['frac'])
for k,o in d['ops'].items(): print(k, o['us'], o['frac_roofline'])
print({k:(v.get('samples_per_s'), v.get('ms_per_forward')) for k,v in d['nets'].items()})
PY
