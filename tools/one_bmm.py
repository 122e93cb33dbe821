"""BERT-large attention Q K^T as one batched GMM launch (B=8, S=512, 16 heads), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

B, S, nh, dh = 8, 512, 16, 64
dev = torch.device("cuda:0")
qkv = torch.randn(B * S, 3 * nh * dh, device=dev).half()
kt = torch.randn(nh * dh, B * S, device=dev).half()
out = torch.empty(B * nh * S, S, device=dev).half()
for _ in range(4):
    tb.gmm_batched(qkv, kt, out, S, S, dh, (B, nh), a=((0, S, 0), (0, 0, dh)), b=((0, 0, dh), (0, S, 0)),
                   c=((0, nh * S, S), (0, 0, 0)))
torch.cuda.synchronize()
