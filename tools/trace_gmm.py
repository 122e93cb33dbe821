"""clock64 trace of CTA 0 of one GMM launch (stage / epilogue timeline) + graph time."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

L = tb.lib()
L.tir_b200_debug_set_trace.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda:0")
buf = torch.zeros(8192, dtype=torch.int64, device=dev)


def graph_us(fn, n=20):
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
    return e0.elapsed_time(e1) / n * 1e3


def show(label, fn):
    us = graph_us(fn)
    buf.zero_()
    torch.cuda.synchronize()
    L.tir_b200_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    fn()
    torch.cuda.synchronize()
    L.tir_b200_debug_set_trace(None)
    t = buf.cpu().tolist()
    t0 = t[1023]
    print(f"== {label}: {us:.1f} us/launch in graph")
    for it in range(12):
        pe, pi, mf, mc = t[2 * it], t[2 * it + 1], t[256 + 2 * it], t[257 + 2 * it]
        if pe == 0 and mf == 0:
            break
        print("stage %3d  prod_wait_done %7d  prod_issued %7d  mma_full %7d  mma_commit %7d" % (it, pe - t0, pi - t0, mf - t0, mc - t0))
    for i in range(12):
        a, b = t[512 + 2 * i], t[513 + 2 * i]
        if a == 0:
            break
        print("tile %2d  epi_start %7d  epi_done %7d" % (i, a - t0, b - t0))
    ctas = [(t[2048 + 4 * i], t[2049 + 4 * i], t[2050 + 4 * i], t[2051 + 4 * i]) for i in range(1024)]
    ctas = [c for c in ctas if c[0]]
    if ctas:
        t0g = min(c[0] for c in ctas)
        ends = sorted(c[1] - t0g for c in ctas)
        print(f"grid {len(ctas)}: end min {ends[0]} median {ends[len(ends)//2]} max {ends[-1]} ns")


M = int(sys.argv[1]) if len(sys.argv) > 1 else 100352
KN = [tuple(map(int, a.split("x"))) for a in sys.argv[2:]] or [(64, 64), (64, 256), (256, 64)]
for K, N in KN:
    A = torch.randn(M, K, device=dev).half()
    B = torch.randn(K, N, device=dev).half()
    bias = torch.randn(N, device=dev)
    R = torch.randn(M, N, device=dev).half()
    C32 = torch.empty(M, N, device=dev)
    C16 = torch.empty(M, N, device=dev).half()
    show(f"M{M} K{K} N{N} f32 plain", lambda: tb.gmm(A, B, C32))
    show(f"M{M} K{K} N{N} f16 plain", lambda: tb.gmm(A, B, C16, out_f16=True))
    show(f"M{M} K{K} N{N} f32 bias+relu", lambda: tb.gmm(A, B, C32, bias=bias, relu=True))
    show(f"M{M} K{K} N{N} f16 relu", lambda: tb.gmm(A, B, C16, out_f16=True, relu=True))
    show(f"M{M} K{K} N{N} f16 bias+relu", lambda: tb.gmm(A, B, C16, out_f16=True, bias=bias, relu=True))
    show(f"M{M} K{K} N{N} f16 bias+res+relu", lambda: tb.gmm(A, B, C16, out_f16=True, bias=bias, relu=True, residual=R))
    show(f"M{M} K{K} N{N} f16 bias+relu6", lambda: tb.gmm(A, B, C16, out_f16=True, bias=bias, relu="relu6"))
