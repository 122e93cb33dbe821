for rep in 1 2; do for lib in ab/lib_base.so ab/lib_bnepi.so; do TIR_B200_LIB=$lib timeout 900 python bench.py --no-cpu --no-e2e --no-ops --nets bert_large 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', {k:v.get('samples_per_s') for k,v in d['nets'].items()})"; done; done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
