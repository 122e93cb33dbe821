# interleaved A/B of an env setting on one op: bash tools/ab_env.sh OP "ENV=VAL" ["ENV2=VAL2"]
OP=$1; shift
for rep in 1 2; do
  for e in "TIR_B200_NOOP=1" "$@"; do
    env $e python bench.py --op $OP --no-ops --no-cpu --no-e2e --no-nets --steps 200 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', '$OP', round(d['ms_per_step']*1e3,3), 'us', d['roofline']['frac'])"
  done
done
