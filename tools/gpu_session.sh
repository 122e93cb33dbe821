timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_epilogue.py -m gpu -x -q -k "gp16 or gp32 or group_packed or narrow or s1d or GRP" 2>&1 | tail -15
