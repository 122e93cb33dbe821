for rep in 1 2 3; do for lib in ab/lib_base2.so ab/lib_wr.so; do for op in C2D DIL; do
TIR_B200_LIB=$lib timeout 300 python bench.py --op $op --no-ops --no-cpu --no-e2e --no-nets --steps 200 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', '$op', round(d['ms_per_step']*1e3,3))"
done; done; done
