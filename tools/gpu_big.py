"""Tensor-bound shapes from SURVEY §8(d): GMM 8192^3 and C2D 14x14x256 (ResNet-50 layer3).
Parity on sampled rows / images vs the oracle (reference distribution), device time via CUDA graph."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2207_04296_b200 as tb
from oracle import oracle as O
from oracle.ir_gen import ConvSpec

dev = torch.device("cuda:0")

def timeit(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for _ in range(n): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e-3

for M, N, K in [(8192, 8192, 8192), (4096, 4096, 4096), (2048, 2048, 2048)]:
    A = torch.from_numpy(O.reference_tensor((M, K), 1)).to(dev).half()
    B = torch.from_numpy(O.reference_tensor((K, N), 2)).to(dev).half()
    C = tb.gmm(A, B); torch.cuda.synchronize()
    rows = [0, M // 2, M - 1]
    a = A.float().cpu().numpy(); b = B.float().cpu().numpy()
    ok = all(O.tensors_bitwise_equal(C[r:r+1].cpu().numpy(), O.gmm(a[r:r+1], b, threads=16)) for r in rows)
    t = timeit(lambda: tb.gmm(A, B, C), n=10 if M >= 8192 else 20)
    print(json.dumps({"case": f"gmm_{M}x{N}x{K}", "exact_rows": ok, "us": round(t * 1e6, 1), "tflops": round(2 * M * N * K / t / 1e12, 1)}), flush=True)

for ci, hw in [(256, 14), (128, 28), (512, 7)]:
    spec = tb.Conv("C2D", n=16, in_dhw=(1, hw, hw), ci=ci, co=ci, k=(1, 3, 3), p=(0, 1, 1))
    X = O.reference_tensor(spec.x_shape(), 3); W = O.reference_tensor(spec.w_shape(), 4)
    Xd = torch.from_numpy(X).to(dev).half(); Wd = torch.from_numpy(W).to(dev).half()
    Y = tb.conv(spec, Xd, Wd); torch.cuda.synchronize()
    o1 = ConvSpec("C2D", n=1, in_dhw=(1, hw, hw), ci=ci, co=ci, k=(1, 3, 3), p=(0, 1, 1))
    ok = O.tensors_bitwise_equal(Y[:1].cpu().numpy(), O.conv(o1, X[:1], W, threads=16))
    t = timeit(lambda: tb.conv(spec, Xd, Wd, Y))
    fl = 2 * tb.useful_macs(spec)
    print(json.dumps({"case": f"c2d_n16_{hw}x{hw}x{ci}", "exact_img0": ok, "us": round(t * 1e6, 2), "tflops": round(fl / t / 1e12, 1)}), flush=True)
