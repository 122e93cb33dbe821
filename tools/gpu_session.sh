timeout 900 python -m pytest tests/test_gpu_epilogue.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_nets.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-ops --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:(v.get('samples_per_s'), v.get('ms_per_forward')) for k,v in d['nets'].items()})"
