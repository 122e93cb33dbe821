"""Wave-quantisation probe for the halo C2D kernel: the paper shape at N = 12..16
images (336..448 tiles of 2 x 56 pixels) and at capped grids, graph-timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

dev = torch.device("cuda:0")


def t_graph(fn, n=100):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n * 1e3, 2)


base = tb.PAPER_SHAPES["C2D"]
for n in (8, 12, 13, 14, 15, 16, 17):
    spec = base.with_(n=n)
    x = torch.randn(spec.x_shape(), device=dev).half()
    w = torch.randn(spec.w_shape(), device=dev).half()
    y = torch.empty(spec.y_shape(), device=dev)
    for cap in (None, 112, 74):
        if cap:
            os.environ["TIR_B200_MAX_CTAS"] = str(cap)
        else:
            os.environ.pop("TIR_B200_MAX_CTAS", None)
        us = t_graph(lambda: tb.conv(spec, x, w, Y=y))
        print(f"N={n:2d} tiles={n * 28} grid={cap or 148}: {us} us", flush=True)
os.environ.pop("TIR_B200_MAX_CTAS", None)
