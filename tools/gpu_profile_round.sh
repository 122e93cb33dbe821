# ncu evidence for profiles/ (round tag $1, default r01):
#  * launch list of the bench headline command (cold-cache, serialised: shares, not absolutes)
#  * one --set full capture per operator family + a ResNet-50 epilogue-bound GEMM + BERT's batched GEMM
TAG=${1:-r01}
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 20 --warmup 3 --no-ops --no-cpu --no-e2e --no-nets > gpurun_out/${TAG}_launches_bench.log 2>&1
for op in C2D GMM DEP C1D GRP T2D DIL C3D; do
  ncu --set full --clock-control none --import-source on -k regex:"igemm|halo|dep_" -s 3 -c 1 \
      -o gpurun_out/${TAG}_full_$op python bench.py --profile $op --steps 2 --warmup 3 > gpurun_out/${TAG}_full_$op.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"igemm" -s 2 -c 1 \
    -o gpurun_out/${TAG}_full_R50_1x1res python tools/one_gmm.py 100352 64 256 f16_bias_relu_res > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"igemm" -s 2 -c 1 \
    -o gpurun_out/${TAG}_full_BERT_qk python tools/one_bmm.py > /dev/null 2>&1
# the cta_group::2 GEMM pairs: the 8192^3 sweep line and BERT-large's FFN1 shape
ncu --set full --clock-control none --import-source on -k regex:"igemm" -s 2 -c 1 \
    -o gpurun_out/${TAG}_full_GMM8K python tools/one_gmm.py 8192 8192 8192 f32 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"igemm" -s 2 -c 1 \
    -o gpurun_out/${TAG}_full_BERT_ffn1 python tools/one_gmm.py 4096 1024 4096 f16_bias > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
# summarise on the box (the reports are ~12 MB each; only C2D's travels back)
python tools/ncu_summary.py ${TAG} > gpurun_out/${TAG}_ncu_summary.txt 2>&1
mkdir -p gpurun_out/profiles_${TAG}
cp profiles/${TAG}_ncu_full_summary.json profiles/ncu_traffic.json gpurun_out/profiles_${TAG}/
for r in gpurun_out/${TAG}_full_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page details --csv > gpurun_out/profiles_${TAG}/${b#${TAG}_full_}_details.csv 2>/dev/null
  ncu -i $r --page source --csv > gpurun_out/profiles_${TAG}/${b#${TAG}_full_}_source.csv 2>/dev/null
done
cp gpurun_out/${TAG}_launches.csv gpurun_out/profiles_${TAG}/
for r in gpurun_out/${TAG}_full_*.ncu-rep; do case $r in *_C2D.ncu-rep) ;; *) rm -f $r ;; esac; done
du -sh gpurun_out
