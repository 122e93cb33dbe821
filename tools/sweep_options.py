"""Sweep planner-switch combinations on bench.py shapes (graph replay, rotating
sets > 2x L2, same timing as bench.py); prints the median us per (op, combo).

  python tools/sweep_options.py --ops T2D,C1D "bn=128,ksplit=8" "bn=64,ksplit=8" ...
The empty combo "" is the default plan.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2207_04296_b200 as tb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("combos", nargs="*", help='"name=value,name=value" per variant')
    ap.add_argument("--ops", default="T2D")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    combos = [""] + a.combos
    parsed = [dict((k, int(v)) for k, v in (s.split("=") for s in c.split(",") if s)) for c in combos]
    names = sorted({k for c in parsed for k in c})
    base = {k: tb.get_option(k) for k in names}
    for op in a.ops.split(","):
        r = bench.OpRunner(op, dev)
        t = {i: [] for i in range(len(combos))}
        for _ in range(a.rounds):
            for i, c in enumerate(parsed):
                for k, x in base.items():
                    tb.set_option(k, x)
                for k, x in c.items():
                    tb.set_option(k, x)
                try:
                    ms, _, _ = bench.time_graph(r, a.steps, 3, None, None)
                    t[i].append(ms / a.steps * 1e3)
                except Exception as e:  # an unsupported plan
                    t[i].append(float("nan"))
                    print(json.dumps({"op": op, "combo": combos[i], "error": str(e)[:200]}), flush=True)
        for k, x in base.items():
            tb.set_option(k, x)
        for i in t:
            print(json.dumps({"op": op, "combo": combos[i] or "default",
                              "us": round(statistics.median(t[i]), 3)}), flush=True)
        del r
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
