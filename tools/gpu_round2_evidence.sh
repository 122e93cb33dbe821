# Round-2 evidence run on the GPU box (outputs under gpurun_out/r02/):
#  * compute-sanitizer memcheck / racecheck / synccheck over one small launch of every kernel family
#  * steady-state DRAM traffic and time per launch of every bench op: ncu profiles one CUDA graph of
#    30 consecutive launches as a single result (--graph-profiling graph; rotating buffers > 2x L2,
#    PDL edges, clocks not locked), so write-backs of earlier launches are counted and the per-launch
#    time includes the PDL overlap
set -x
mkdir -p gpurun_out/r02
for tool in ${SANITIZERS-memcheck racecheck synccheck}; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py \
      > gpurun_out/r02/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r02/sanitizer_$tool.txt
done
for op in ${OPS:-C2D GMM C1D GRP T2D DEP DIL C3D DEP_112c96s2 DEP_56c144s1 GMM8K C2D_L3}; do
  steps=30; case $op in C3D|GMM8K) steps=6;; esac
  timeout 600 ncu --graph-profiling graph --profile-from-start off --cache-control none --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
      python bench.py --profile-range $op --steps $steps --warmup 3 > gpurun_out/r02/range_$op.csv 2> gpurun_out/r02/range_$op.err
  rc=$?
  steps=$(grep -o '"launches": [0-9]*' gpurun_out/r02/range_$op.csv | grep -o '[0-9]*$')
  echo "$op rc=$rc steps=$steps" >> gpurun_out/r02/range_steps.txt
done
tail -3 gpurun_out/r02/range_C2D.csv
