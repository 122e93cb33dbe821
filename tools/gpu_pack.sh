for c in dil_small c3d_small dil_paper c2d_ci8; do python tests/gpu_diag.py $c; done > gpurun_out/pack.txt 2>&1
python -m pytest tests/test_gpu_parity.py -q -k "DIL or C3D or dil or c3d" --timeout 900 2>&1 | tail -2 >> gpurun_out/pack.txt
python bench.py --op DIL --steps 100 --warmup 3 --no-ops --no-cpu --no-e2e > gpurun_out/dil_bench.json 2>/dev/null
python bench.py --op C3D --steps 10 --warmup 3 --no-ops --no-cpu --no-e2e > gpurun_out/c3d_bench.json 2>/dev/null
