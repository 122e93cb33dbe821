for op in T2D GRP; do timeout 120 python tools/cta_timeline.py $op 4 2>&1 | sed -n 2,3p; done
