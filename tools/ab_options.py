"""In-process A/B of libtir_b200 planner switches (tir_b200_set_option) on the
bench.py sweep shapes: the same graph-replay timing as bench.py (rotating sets >
2x L2), alternating A and B runs to cancel drift; prints the median us per op.

  python tools/ab_options.py l2_prefetch=0 [mc=0 ...] [--ops C2D,GMM] [--rounds 3]
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
    ap.add_argument("switches", nargs="+", help="name=value (applied together as variant B)")
    ap.add_argument("--ops", default="GMM,C1D,C2D,DIL,GRP,T2D,DEP,DEP_112c96s2,DEP_56c144s1,C2D_L3")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    sw = dict((k, int(v)) for k, v in (s.split("=") for s in a.switches))
    base = {k: tb.get_option(k) for k in sw}
    res = {}
    for op in a.ops.split(","):
        r = bench.OpRunner(op, dev)
        t = {"A": [], "B": []}
        for _ in range(a.rounds):
            for v, vals in (("A", base), ("B", sw)):
                for k, x in vals.items():
                    tb.set_option(k, x)
                ms, _, _ = bench.time_graph(r, a.steps, 3, None, None)
                t[v].append(ms / a.steps * 1e3)
        for k, x in base.items():
            tb.set_option(k, x)
        res[op] = {"A_us": round(statistics.median(t["A"]), 3), "B_us": round(statistics.median(t["B"]), 3)}
        print(json.dumps({"op": op, "B": sw, **res[op]}), flush=True)
        del r
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
