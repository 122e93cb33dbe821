"""Event-timed GMM (fp16 in, fp32 out) of one shape: python tools/time_gmm.py M K N [iters].
Quick A/B of host env knobs (TIR_B200_KS, TIR_B200_BN ...) without the bench harness."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 20
dev = torch.device("cuda:0")
A = torch.randn(M, K, device=dev).half()
B = torch.randn(K, N, device=dev).half()
C = torch.empty(M, N, device=dev, dtype=torch.float32)
for _ in range(3):
    tb.gmm(A, B, C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    tb.gmm(A, B, C)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / iters
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("TIR_B200_"))
print(f"{env or 'default'} {M}x{K}x{N}: {us:.1f} us  {2 * M * N * K / us / 1e6:.0f} TFLOPS", flush=True)
