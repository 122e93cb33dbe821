mkdir -p gpurun_out/s6
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s6/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/s6/pytest_gpu.txt
export TIR_B200_L2_PREFETCH=2
python tools/cta_timeline.py C2D 4 > gpurun_out/s6/cta.txt 2>&1
cat gpurun_out/s6/cta.txt
for op in C2D C2D_L3; do python bench.py --op $op --no-cpu --no-e2e --no-nets --no-ops --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$op', d['ms_per_step']*1e3, d['roofline']['frac'])"; done
