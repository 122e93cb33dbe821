"""Where the headline e2e step goes (bench.py measure_e2e, tir_b200_conv_host): the
synchronous host-buffer call next to a copy-only pipeline of the same chunking (H2D
chunks on one stream, D2H chunks on another, each D2H after its chunk's H2D), host
wall clock, median of 30 calls."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2207_04296_b200 as tb  # noqa: E402


def med(fn, n=30):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6


spec = bench.op_spec("C2D")
rng = np.random.default_rng(7)
X = torch.from_numpy(rng.standard_normal(spec.x_shape(), dtype=np.float32).astype(np.float16)).pin_memory()
W = torch.from_numpy(rng.standard_normal(spec.w_shape(), dtype=np.float32).astype(np.float16)).pin_memory()
Y = torch.empty(spec.y_shape(), dtype=torch.float32).pin_memory()
Xn, Wn, Yn = X.numpy(), W.numpy(), Y.numpy()
print("conv_host us", round(med(lambda: tb.conv_host(spec, Xn, Wn, Yn)), 1))
dX, dY = torch.empty_like(X, device="cuda"), torch.empty_like(Y, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for chunks in (1, 4, 8, 16):
    evs = [torch.cuda.Event() for _ in range(chunks)]

    def pipe():
        n = X.shape[0]
        for c in range(chunks):
            a, b = n * c // chunks, n * (c + 1) // chunks
            with torch.cuda.stream(s1):
                dX[a:b].copy_(X[a:b], non_blocking=True)
                evs[c].record(s1)
            s2.wait_event(evs[c])
            with torch.cuda.stream(s2):
                Y[a:b].copy_(dY[a:b], non_blocking=True)
        s2.synchronize()
    print(f"copy-only pipeline, {chunks} chunks, us", round(med(pipe), 1))

# inside the C-ABI call: enqueue time vs total (tir_b200_debug_host_times)
import ctypes  # noqa: E402

L = tb.lib()
L.tir_b200_debug_host_times.argtypes = [ctypes.POINTER(ctypes.c_double)]
buf = (ctypes.c_double * 2)()
enq, tot = [], []
for _ in range(30):
    tb.conv_host(spec, Xn, Wn, Yn)
    L.tir_b200_debug_host_times(buf)
    enq.append(buf[0])
    tot.append(buf[1])
print("inside conv_host: enqueue us", round(statistics.median(enq), 1), "total us", round(statistics.median(tot), 1))

# the bare ctypes call with precomputed arguments vs the Python wrapper
d = spec.desc()
px, pw, py = ctypes.c_void_p(Xn.ctypes.data), ctypes.c_void_p(Wn.ctypes.data), ctypes.c_void_p(Yn.ctypes.data)
print("bare ctypes call us", round(med(lambda: L.tir_b200_conv_host(ctypes.byref(d), px, pw, py, 0)), 1))
print("wrapper prep only us", round(med(lambda: (spec.desc(), np.ascontiguousarray(Xn), np.ascontiguousarray(Wn),
                                                  ctypes.c_void_p(Xn.ctypes.data))), 1))
