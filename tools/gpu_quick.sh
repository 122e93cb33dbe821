# quick iteration on the GPU box: full GPU tests, then the headline op timed
# (graph replay, L2-rotating buffers) with and without an env toggle.
# usage: bash tools/gpu_quick.sh [ENV_TOGGLE] [OP...]
TOGGLE=${1:-TIR_B200_NOOP}
shift
OPS=${@:-C2D}
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.txt
for op in $OPS; do
  timeout 120 python bench.py --op $op --no-ops --no-cpu --no-e2e --steps 200 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$op', 'default', d['ms_per_step']*1e3, 'us', d['roofline']['frac'])"
  env $TOGGLE=1 timeout 120 python bench.py --op $op --no-ops --no-cpu --no-e2e --steps 200 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$op', '$TOGGLE', d['ms_per_step']*1e3, 'us', d['roofline']['frac'])"
done
