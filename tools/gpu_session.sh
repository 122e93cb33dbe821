mkdir -p gpurun_out/s17
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rowpack or C3D or stem" > gpurun_out/s17/pytest_rp.txt 2>&1; rc=$?; echo "pytest rc=$rc"
tail -1 gpurun_out/s17/pytest_rp.txt
timeout 300 python bench.py --op C3D --no-cpu --no-e2e --no-nets --no-ops --steps 10 2>gpurun_out/s17/bench_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3D', d['ms_per_step']*1e3, d['value'], d['roofline']['frac'])"
timeout 120 python tools/cta_timeline.py C3D 2 2>&1 | tail -6
