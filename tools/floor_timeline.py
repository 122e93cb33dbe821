"""Per-launch floor breakdown from %globaltimer milestones (igemm.cuh trace_event).

Captures K back-to-back launches of one bench.py op in a CUDA graph (PDL edges,
as in bench.py), each launch with its own trace buffer, replays it, and prints
for the launches in the middle of the sequence (ns, medians):
  period           exit(k-1) -> exit(k): the steady-state time per launch
  entry_vs_prev    entry(k) - exit(k-1) (negative: PDL started the CTA early)
  wait             entry -> griddepcontrol.wait returned in the producer
  first_tma        wait returned -> first full barrier (first operand stage landed)
  mma              first full -> first accumulator published (tfull)
  epilogue         tfull -> all TMA stores complete
  tail             stores complete -> kernel exit
Usage: python tools/floor_timeline.py [OP ...]  (bench.py op names; FLOOR = the one-CTA GEMM)
(The relayout kernels of DIL / C3D carry no trace; their conv kernel does.)
"""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2207_04296_b200 as tb  # noqa: E402

EV = ["entry", "pdl_done", "first_full", "first_tfull", "stores_done", "exit"]


def timeline(op, launches=12, reps=5):
    """op: a bench.py op name (rotating buffer sets as in bench.py)."""
    dev = torch.device("cuda:0")
    L = tb.lib()
    L.tir_b200_debug_set_trace.argtypes = [ctypes.c_void_p]
    r = bench.OpRunner(op, dev)
    bufs = [torch.zeros(16384, dtype=torch.int64, device=dev) for _ in range(launches)]
    for i in range(3):
        r.step(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for i in range(launches):
            L.tir_b200_debug_set_trace(bufs[i].data_ptr())
            r.step(i)
    L.tir_b200_debug_set_trace(None)
    rows = {k: [] for k in ("period", "entry_vs_prev", "wait", "first_tma", "mma", "epilogue", "tail")}
    for _ in range(reps):
        for b in bufs:
            b.zero_()
        g.replay()
        torch.cuda.synchronize()
        tl = []
        for b in bufs:
            t = b[8192:8192 + 8 * 256].view(256, 8)[:, :6].cpu()
            used = t[:, 0] > 0
            t = t[used]
            if t.shape[0] == 0:
                tl.append(None)
                continue
            tl.append({"entry": int(t[:, 0].min()), "pdl_done": int(t[:, 1].max()),
                       "first_full": int(t[:, 2].max()), "first_tfull": int(t[:, 3].max()),
                       "stores_done": int(t[:, 4].max()), "exit": int(t[:, 5].max()), "ctas": int(used.sum())})
        for k in range(2, launches - 1):
            p, c = tl[k - 1], tl[k]
            if p is None or c is None:
                continue
            rows["period"].append(c["exit"] - p["exit"])
            rows["entry_vs_prev"].append(c["entry"] - p["exit"])
            rows["wait"].append(c["pdl_done"] - c["entry"])
            rows["first_tma"].append(c["first_full"] - c["pdl_done"])
            rows["mma"].append(c["first_tfull"] - c["first_full"])
            rows["epilogue"].append(c["stores_done"] - c["first_tfull"])
            rows["tail"].append(c["exit"] - c["stores_done"])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    out = {k: statistics.median(v) for k, v in rows.items()}
    out["graph_us_per_launch_traced"] = round(e0.elapsed_time(e1) * 1e3 / launches, 3)
    out["ctas"] = tl[-1]["ctas"]
    return out


if __name__ == "__main__":
    ops = sys.argv[1:] or ["FLOOR", "GMM", "C1D", "C2D", "GRP", "T2D", "DIL"]
    for op in ops:
        print(json.dumps({"op": op, **timeline(op)}), flush=True)
