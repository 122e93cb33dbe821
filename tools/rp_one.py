"""Debug aid: one rowpack conv launch of a given shape (no oracle)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

d, h, w, n = (int(v) for v in sys.argv[1:5])
spec = tb.Conv("C3D", n=n, in_dhw=(d, h, w), ci=3, co=64, k=(7, 7, 7), s=(2, 2, 2), p=(3, 3, 3))
x = torch.randn(*spec.x_shape(), device="cuda").half()
wt = torch.randn(*spec.w_shape(), device="cuda").half()
y = tb.conv(spec, x, wt)
torch.cuda.synchronize()
print("ran", spec.in_dhw, float(y.abs().sum()))
