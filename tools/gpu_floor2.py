"""Per-launch floor inside a CUDA graph: tiny problems of each kernel family, with
the library's knobs toggled in-process (PDL, simple DEP kernel)."""
import json
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


A = torch.randn(128, 64, device=dev).half(); B = torch.randn(64, 64, device=dev).half(); C = torch.empty(128, 64, device=dev)
s1 = tb.Conv("DEP", n=1, in_dhw=(1, 8, 32), ci=32, co=32, k=(1, 3, 3), p=(0, 1, 1), groups=32)
X = torch.randn(*s1.x_shape(), device=dev).half(); W = torch.randn(*s1.w_shape(), device=dev).half(); Y = torch.empty(*s1.y_shape(), device=dev)
x = torch.empty(1, device=dev)
p = tb.PAPER_SHAPES["DEP"]
PX = torch.randn(*p.x_shape(), device=dev).half(); PW = torch.randn(*p.w_shape(), device=dev).half(); PY = torch.empty(*p.y_shape(), device=dev)
for env in ({}, {"TIR_B200_NO_PDL": "1"}, {"TIR_B200_DEP_SIMPLE": "1"}):
    for k, v in env.items():
        os.environ[k] = v
    r = {"env": env,
         "gmm_128x64x64": t_graph(lambda: tb.gmm(A, B, C)),
         "dep_1block": t_graph(lambda: tb.conv(s1, X, W, Y)),
         "dep_paper": t_graph(lambda: tb.conv(p, PX, PW, PY), 20),
         "torch_fill": t_graph(lambda: x.fill_(1.0))}
    print(json.dumps(r), flush=True)
    for k in env:
        del os.environ[k]
