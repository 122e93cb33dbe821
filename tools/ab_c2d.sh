# interleaved A/B of the headline op between two library builds: bash tools/ab_c2d.sh A.so B.so [op]
OP=${3:-C2D}
for rep in 1 2 3; do
  for lib in $1 $2; do
    TIR_B200_LIB=$lib python bench.py --op $OP --no-ops --no-cpu --no-e2e --no-nets --steps 200 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)', '$OP', round(d['ms_per_step']*1e3,3), 'us')"
  done
done
