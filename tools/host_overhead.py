"""CPU cost per C-ABI call of the headline conv (device pointers, async): the host
work of planning (tensor-map encodes, function attributes, launch) per call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

spec = tb.PAPER_SHAPES["C2D"]
for n in (16, 2):
    s = spec.with_(n=n)
    x = torch.randn(*s.x_shape(), device="cuda").half()
    w = torch.randn(*s.w_shape(), device="cuda").half()
    y = torch.empty(*s.y_shape(), device="cuda")
    for _ in range(20):
        tb.conv(s, x, w, y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        tb.conv(s, x, w, y)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"n={n}: {1e6 * (t1 - t0) / 200:.1f} us CPU per tb.conv call (python + C-ABI)")
