"""Per-launch floor of each kernel family inside a CUDA graph (tiny problems)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2207_04296_b200 as tb
dev = torch.device("cuda:0")

def t_graph(fn, n=50):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for _ in range(n): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3

A = torch.randn(128, 64, device=dev).half(); B = torch.randn(64, 64, device=dev).half(); C = torch.empty(128, 64, device=dev)
print(json.dumps({"case": "gmm_128x64x64 (1 CTA, 1 stage)", "us": round(t_graph(lambda: tb.gmm(A, B, C)), 2)}))
A2 = torch.randn(128, 1024, device=dev).half(); B2 = torch.randn(1024, 64, device=dev).half(); C2 = torch.empty(128, 64, device=dev)
print(json.dumps({"case": "gmm_128x64x1024 (1 CTA, 4 stages)", "us": round(t_graph(lambda: tb.gmm(A2, B2, C2)), 2)}))
spec = tb.Conv("C2D", n=1, in_dhw=(1, 8, 8), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1))
X = torch.randn(*spec.x_shape(), device=dev).half(); W = torch.randn(*spec.w_shape(), device=dev).half(); Y = torch.empty(*spec.y_shape(), device=dev)
print(json.dumps({"case": "halo c2d 8x8x64 (1 tile)", "us": round(t_graph(lambda: tb.conv(spec, X, W, Y)), 2)}))
spec = tb.Conv("DEP", n=1, in_dhw=(1, 8, 32), ci=32, co=32, k=(1, 3, 3), p=(0, 1, 1), groups=32)
X = torch.randn(*spec.x_shape(), device=dev).half(); W = torch.randn(*spec.w_shape(), device=dev).half(); Y = torch.empty(*spec.y_shape(), device=dev)
print(json.dumps({"case": "dep 8x32x32 (1 block)", "us": round(t_graph(lambda: tb.conv(spec, X, W, Y)), 2)}))
x = torch.empty(1, device=dev)
print(json.dumps({"case": "torch fill_ (empty-ish kernel)", "us": round(t_graph(lambda: x.fill_(1.0)), 2)}))
os.environ["TIR_B200_NO_PDL"] = "1"
