"""One GMM configuration launched a few times (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

M, K, N, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
dev = torch.device("cuda:0")
A = torch.randn(M, K, device=dev).half()
B = torch.randn(K, N, device=dev).half()
bias = torch.randn(N, device=dev)
R = torch.randn(M, N, device=dev).half()
C = torch.empty(M, N, device=dev, dtype=torch.float32 if mode.startswith("f32") else torch.float16)
kw = dict(out_f16=not mode.startswith("f32"))
if "bias" in mode:
    kw["bias"] = bias
if "relu" in mode:
    kw["relu"] = True
if "res" in mode:
    kw["residual"] = R
for _ in range(4):
    tb.gmm(A, B, C, **kw)
torch.cuda.synchronize()
