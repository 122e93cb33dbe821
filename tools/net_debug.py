"""Runs a network graph op by op with a synchronize after each (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2207_04296_b200 import api, nets  # noqa: E402

name, batch, image = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
net = nets.NETS[name](batch, image=image)
dn = nets.DeviceNet(net, torch.device("cuda:0"))
dn.input.normal_()
ops = net.ops
for i, op in enumerate(ops):
    try:
        with torch.cuda.stream(dn.stream):
            dn.run(i, i + 1)
        torch.cuda.synchronize()
    except Exception as e:
        print("FAIL", i, op.kind, op.spec, op.w.shape if op.w is not None else None, net.shapes[op.src],
              net.shapes[op.dst], op.act, op.res, repr(e)[:300])
        sys.exit(1)
print("all ok", len(ops))
