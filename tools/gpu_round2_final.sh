# Round-2 final evidence (outputs under gpurun_out/r02f/, summaries copied to profiles/ by the builder):
#  * compute-sanitizer memcheck / racecheck / synccheck over every kernel family (incl. conv_rowpack_kernel)
#  * ncu --set full of one launch per kernel family at the paper shapes (details + source pages)
#  * steady-state DRAM traffic per launch of every bench op (graph profiling, rotating buffers > 2x L2)
#  * the launch list of the headline bench command
T=gpurun_out/r02f
mkdir -p $T
for tool in ${SANITIZERS-memcheck racecheck synccheck}; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > $T/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -2 $T/sanitizer_$tool.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $T/launches_bench_c2d.csv \
    python bench.py --steps 20 --warmup 3 --no-ops --no-cpu --no-e2e --no-nets > $T/launches_bench.log 2>&1
for op in ${FULL_OPS:-C2D C3D DIL GMM C1D GRP T2D DEP}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"igemm|halo|dep_|conv_rowpack" -s 3 -c 1 \
      -o $T/full_$op python bench.py --profile $op --steps 2 --warmup 3 > $T/full_$op.log 2>&1
  ncu -i $T/full_$op.ncu-rep --page details --csv > $T/full_${op}_details.csv 2>/dev/null
  ncu -i $T/full_$op.ncu-rep --page raw --csv > $T/full_${op}_raw.csv 2>/dev/null
  rm -f $T/full_$op.ncu-rep
done
for op in ${OPS:-C2D GMM C1D GRP T2D DEP DIL C3D DEP_112c96s2 DEP_56c144s1 GMM8K C2D_L3}; do
  steps=30; case $op in C3D|GMM8K) steps=6;; esac
  timeout 600 ncu --graph-profiling graph --profile-from-start off --cache-control none --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
      python bench.py --profile-range $op --steps $steps --warmup 3 > $T/range_$op.csv 2> $T/range_$op.err
  rc=$?
  steps=$(grep -o '"launches": [0-9]*' $T/range_$op.csv | grep -o '[0-9]*$')
  echo "$op rc=$rc steps=$steps" >> $T/range_steps.txt
done
du -sh $T
