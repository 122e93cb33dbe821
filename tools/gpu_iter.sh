# quick iteration: kernel trace, parity sweep, bench (no CPU leg)
python tools/trace_igemm.py > gpurun_out/trace.txt 2>&1
python tests/gpu_diag.py > gpurun_out/diag.txt 2>&1
python bench.py --steps 200 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
