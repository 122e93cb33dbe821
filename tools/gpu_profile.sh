# ncu evidence for profiles/: per-launch device times of the bench command and
# one --set full capture per kernel family (cold-cache, serialised replays).
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r01_launches.csv \
    python bench.py --steps 20 --warmup 3 --no-ops --no-cpu --no-e2e > gpurun_out/r01_launches_bench.log 2>&1
for op in C2D GMM DEP GRP T2D C1D; do
  ncu --set full --clock-control none --import-source on -k regex:"igemm|halo|dep_" -s 3 -c 1 \
      -o gpurun_out/r01_full_$op python bench.py --profile $op --steps 2 --warmup 3 > gpurun_out/r01_full_$op.log 2>&1
done
ls -la gpurun_out
