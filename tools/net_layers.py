"""Per-op device time of a network graph: each op captured alone in a CUDA graph
of 20 launches and replayed between CUDA events (debug / tuning aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2207_04296_b200 import nets  # noqa: E402

name, batch = sys.argv[1], int(sys.argv[2])
net = nets.NETS[name](batch)
dn = nets.DeviceNet(net, torch.device("cuda:0"))
dn.input.normal_()
with torch.cuda.stream(dn.stream):
    dn.run()
torch.cuda.synchronize()
rows = []
total = 0.0
for i, op in enumerate(net.ops):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(dn.stream):
        dn.run(i, i + 1)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=dn.stream, capture_error_mode="relaxed"):
        for _ in range(20):
            dn.run(i, i + 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(dn.stream):
        g.replay()
        e0.record(dn.stream)
        g.replay()
        e1.record(dn.stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    total += us
    n, h, w, c = net.shapes[op.src]
    co = net.shapes[op.dst][-1]
    if op.kind in ("conv", "dep"):
        sp = op.spec
        oh, ow = net.shapes[op.dst][1:3]
        fl = 2 * n * oh * ow * co * sp.k[1] * sp.k[2] * (c // sp.groups)
        desc = f"{op.kind} {h}x{w}x{c}->{co} k{sp.k[1]} s{sp.s[1]}"
    elif op.kind == "gmm":
        k, nn = op.w.shape
        m = n * h * w
        fl = 2 * m * k * nn
        desc = f"gmm M{m} K{k} N{nn}"
    else:
        fl = 0
        desc = f"{op.kind} {h}x{w}x{c}"
    byts = (n * h * w * c + torch.tensor(net.shapes[op.dst]).prod().item()) * 2
    print(f"{i:3d} {desc:38s} {us:8.1f} us  {fl / us / 1e6:7.1f} TF  {byts / us / 1e3:7.1f} GB/s"
          f"{' +res' if op.res else ''}", flush=True)
print(f"sum {total:.1f} us")
