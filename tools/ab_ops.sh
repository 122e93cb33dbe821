# A/B of two builds of the library on the op sweep, interleaved (same box, same clocks)
# usage: bash tools/ab_ops.sh OLD_SO [NEW_SO]
OLD=$1; NEW=${2:-paper_2207_04296_b200/lib/libtir_b200.so}
for rep in 1 2; do
  for lib in $OLD $NEW; do
    TIR_B200_LIB=$lib python bench.py --no-cpu --no-e2e --no-nets --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)'[:18], {k:v.get('us') for k,v in d['ops'].items()})"
  done
done
