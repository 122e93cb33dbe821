python tests/gpu_diag.py c2d_paper > gpurun_out/ab.txt 2>&1
TIR_B200_STORE256=1 python tests/gpu_diag.py c2d_paper halo_c2d_wide halo_c2d_co256 >> gpurun_out/ab.txt 2>&1
python bench.py --steps 200 --warmup 5 --no-cpu --no-ops --no-e2e > gpurun_out/ab_default.json 2>/dev/null
TIR_B200_STORE256=1 python bench.py --steps 200 --warmup 5 --no-cpu --no-ops --no-e2e > gpurun_out/ab_s256.json 2>/dev/null
