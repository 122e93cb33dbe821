set -x
python bench.py --steps 200 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2d.csv python bench.py --profile C2D --steps 5 --warmup 3 > /dev/null 2>&1
for op in C2D GMM DEP; do
ncu --set full --clock-control none --import-source on -k regex:"igemm|dep_kernel" -s 3 -c 1 -o gpurun_out/prof_$op python bench.py --profile $op --steps 3 --warmup 3 > gpurun_out/ncu_$op.log 2>&1
done
ls -la gpurun_out
