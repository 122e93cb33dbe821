for c in dep_small dep_paper dep_s2; do python tests/gpu_diag.py $c; done > gpurun_out/dep.txt 2>&1
python -m pytest tests/test_gpu_parity.py -q -k "DEP or dep" --timeout 600 2>&1 | tail -2 >> gpurun_out/dep.txt
python bench.py --op DEP --steps 200 --warmup 5 --no-ops --no-cpu --no-e2e > gpurun_out/dep_bench.json 2>/dev/null
