"""Summarises `ncu --graph-profiling graph` captures of bench.py --profile-range
(tools/gpu_round2_evidence.sh) into profiles/<tag>_ncu_graph_traffic.json:
steady-state DRAM bytes per launch (read + write over a CUDA graph of K
consecutive launches on rotating buffers > 2x L2, so write-backs of earlier
launches are counted) next to the algorithmic bytes of bench.op_work.

  python tools/ncu_graph_summary.py gpurun_out/r02 r02
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main(src, tag):
    steps = {}
    for ln in open(os.path.join(src, "range_steps.txt")):
        f = ln.split()
        steps[f[0]] = int(f[2].split("=")[1])
    out = {}
    for op, k in steps.items():
        path = os.path.join(src, f"range_{op}.csv")
        vals = {}
        with open(path) as fh:
            rows = [r for r in csv.reader(fh) if len(r) > 14 and r[0] != "ID"]
        for r in rows:
            vals[r[12]] = float(r[14].replace(",", ""))
        if "dram__bytes_read.sum" not in vals:
            out[op] = {"error": "no metrics"}
            continue
        f, b, bound = bench.op_work(op)
        rd, wr = vals["dram__bytes_read.sum"] / k, vals["dram__bytes_write.sum"] / k
        out[op] = {"launches_in_graph": k, "dram_read_per_launch": round(rd), "dram_write_per_launch": round(wr),
                   "traffic_per_launch": round(rd + wr), "algorithmic_bytes": b,
                   "traffic_over_algorithmic": round((rd + wr) / b, 3),
                   "ncu_graph_us_per_launch": round(vals.get("gpu__time_duration.sum", 0) / k / 1e3, 3)}
    dst = os.path.join(ROOT, "profiles", f"{tag}_ncu_graph_traffic.json")
    with open(dst, "w") as fh:
        json.dump({"how": "ncu --graph-profiling graph --profile-from-start off --cache-control none "
                          "--clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                          "gpu__time_duration.sum python bench.py --profile-range OP --steps K (one CUDA graph of K "
                          "launches on rotating buffer sets > 2x L2, profiled as one result). ncu serialises the "
                          "graph under its own instrumentation, so its time per launch is an upper bound, not "
                          "the bench number.", "ops": out}, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
