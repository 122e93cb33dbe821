for e in 0 1; do TIR_B200_EPI8=$e timeout 300 python bench.py --op GRP --no-ops --no-cpu --no-e2e --no-nets --steps 200 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('GRP epi8=$e', round(d['ms_per_step']*1e3,3))"; done
TIR_B200_EPI8=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "GRP" 2>&1 | tail -1
