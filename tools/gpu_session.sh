timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/cta_timeline.py DEP 4 2>&1 | grep -v "^  block\|last 6" | head -8
timeout 120 python tools/cta_timeline.py C2D 4 2>&1 | sed -n 2,3p
