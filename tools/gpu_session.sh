for rep in 1 2; do for lib in ab/lib_rp5.so ab/lib_desc2.so; do for op in C3D DIL; do
TIR_B200_LIB=$lib timeout 300 python bench.py --op $op --no-ops --no-cpu --no-e2e --no-nets --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', '$op', round(d['ms_per_step']*1e3,2), d['clocks']['sm_mhz'])"
done; done; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_epilogue.py tests/test_gpu_nets.py -m gpu -x -q -k "rowpack or C3D or stem or DIL or resnet or mobilenet" 2>&1 | tail -1
