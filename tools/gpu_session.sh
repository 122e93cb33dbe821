mkdir -p gpurun_out/s30
timeout 900 python bench.py > gpurun_out/s30/bench.json 2> gpurun_out/s30/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/s30/bench.json').read().strip().splitlines()[-1])
print('headline', d['value'], d['ms_per_step'], d['roofline'], d['clocks'])
print('e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'])
for k,o in d['ops'].items(): print(k, o['us'], o['tflops'], o['gbs'], o['frac_roofline'], o.get('frac_roofline_ex_floor'))
print({k:(v.get('samples_per_s'), v.get('ms_per_forward')) for k,v in d['nets'].items()})
PY
