"""Per-launch floor breakdown from %globaltimer milestones (igemm.cuh trace_event).

Captures K back-to-back launches of one GEMM shape in a CUDA graph (PDL edges,
as in bench.py), each launch with its own trace buffer, replays it, and prints
for the launches in the middle of the sequence (ns, medians):
  period           exit(k-1) -> exit(k): the steady-state time per launch
  entry_vs_prev    entry(k) - exit(k-1) (negative: PDL started the CTA early)
  wait             entry -> griddepcontrol.wait returned in the producer
  first_tma        wait returned -> first full barrier (first operand stage landed)
  mma              first full -> first accumulator published (tfull)
  epilogue         tfull -> all TMA stores complete
  tail             stores complete -> kernel exit
Usage: python tools/floor_timeline.py [M N K ...]  (default: the one-CTA floor GEMM and GMM 1024^3)
"""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

EV = ["entry", "pdl_done", "first_full", "first_tfull", "stores_done", "exit"]


def timeline(M, N, K, launches=12, reps=5):
    dev = torch.device("cuda:0")
    L = tb.lib()
    L.tir_b200_debug_set_trace.argtypes = [ctypes.c_void_p]
    sets = 8
    A = [torch.randn(M, K, device=dev).half() for _ in range(sets)]
    B = [torch.randn(K, N, device=dev).half() for _ in range(sets)]
    C = [torch.empty(M, N, device=dev) for _ in range(sets)]
    bufs = [torch.zeros(16384, dtype=torch.int64, device=dev) for _ in range(launches)]
    for i in range(3):
        tb.gmm(A[i % sets], B[i % sets], C[i % sets])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for i in range(launches):
            L.tir_b200_debug_set_trace(bufs[i].data_ptr())
            tb.gmm(A[i % sets], B[i % sets], C[i % sets])
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
            tl.append({"entry": int(t[:, 0].min()), "pdl_done": int(t[:, 1].max()),
                       "first_full": int(t[:, 2].max()), "first_tfull": int(t[:, 3].max()),
                       "stores_done": int(t[:, 4].max()), "exit": int(t[:, 5].max()), "ctas": int(used.sum())})
        for k in range(2, launches - 1):
            p, c = tl[k - 1], tl[k]
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
    shapes = [(128, 64, 64), (1024, 1024, 1024)]
    if len(sys.argv) > 1:
        a = [int(v) for v in sys.argv[1:]]
        shapes = [tuple(a[i:i + 3]) for i in range(0, len(a), 3)]
    for s in shapes:
        print(json.dumps({"shape": s, **timeline(*s)}), flush=True)
