# A/B of epilogue modes on the C2D headline (bench only)
for mode in default no_tma_store; do
  if [ $mode = no_tma_store ]; then export TIR_B200_NO_TMA_STORE=1; fi
  python bench.py --steps 200 --warmup 5 --no-cpu --no-ops --no-e2e > gpurun_out/ab_$mode.json 2>/dev/null
  TIR_B200_NO_PDL=1 python bench.py --steps 200 --warmup 5 --no-cpu --no-ops --no-e2e > gpurun_out/ab_${mode}_nopdl.json 2>/dev/null
done
python tools/trace_igemm.py > gpurun_out/trace_direct.txt 2>&1
