timeout 120 python tools/cta_timeline.py C3D 2 2>&1 | grep "per-depth" | cut -c1-300
for op in C3D DIL; do timeout 300 python bench.py --op $op --no-ops --no-cpu --no-e2e --no-nets --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$op', round(d['ms_per_step']*1e3,2))"; done
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rowpack or C3D" 2>&1 | tail -1
