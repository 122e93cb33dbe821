"""Per-op device time of one BERT-large encoder layer (B=8, S=512), each op
captured alone in a CUDA graph of 20 launches (tuning aid)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2207_04296_b200 import api, nets  # noqa: E402

net = nets.bert_large(8, layers=1)
dn = nets.device_net(net, torch.device("cuda:0"))
dn.x.normal_()
B, S, H, nh, dh = net.batch, net.seq, net.hidden, net.heads, net.head_dim
w = dn.w[0]
st = dn.stream
T = net.tokens
ops = [
    ("qkv gmm", 2 * T * H * 3 * H, lambda: api.gmm(dn.x, w["w_qkv"], dn.qkv, out_f16=True, bias=w["b_qkv"], stream=st)),
    ("QK^T batched", 2 * B * nh * S * S * dh, lambda: api.gmm_batched(dn.qkv, dn.qkv, dn.scores, S, S, dh, (B, nh),
        a=((0, S, 0), (0, 0, dh)), b=((0, S, 0), (H, 0, dh)), c=((0, nh * S, S), (0, 0, 0)), b_kmajor=True,
        stream=st)),
    ("softmax", 0, lambda: api.softmax(dn.scores, 1 / math.sqrt(dh), Y=dn.scores, stream=st)),
    ("PV batched", 2 * B * nh * S * S * dh, lambda: api.gmm_batched(dn.scores, dn.qkv, dn.ctx, S, dh, S, (B, nh),
        a=((0, nh * S, S), (0, 0, 0)), b=((0, S, 0), (2 * H, 0, dh)), c=((0, S, 0), (0, 0, dh)), stream=st)),
    ("out gmm +res", 2 * T * H * H, lambda: api.gmm(dn.ctx, w["w_o"], dn.attn, out_f16=True, bias=w["b_o"], residual=dn.x, stream=st)),
    ("layernorm", 0, lambda: api.layernorm(dn.attn, w["ln1_g"], w["ln1_b"], net.eps, Y=dn.x1, stream=st)),
    ("ffn1 gmm gelu", 2 * T * H * net.ffn, lambda: api.gmm(dn.x1, w["w_f1"], dn.hid, out_f16=True, bias=w["b_f1"], relu="gelu", stream=st)),
    ("ffn2 gmm +res", 2 * T * H * net.ffn, lambda: api.gmm(dn.hid, w["w_f2"], dn.y, out_f16=True, bias=w["b_f2"], residual=dn.x1, stream=st)),
    ("layernorm", 0, lambda: api.layernorm(dn.y, w["ln2_g"], w["ln2_b"], net.eps, Y=dn.x, stream=st)),
]
total = 0
for name, fl, fn in ops:
    with torch.cuda.stream(st):
        fn()
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
        for _ in range(20):
            fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        g.replay()
        e0.record(st)
        g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    total += us
    print(f"{name:16s} {us:8.1f} us  {fl / us / 1e6 if fl else 0:7.1f} TFLOPS", flush=True)
print(f"layer total {total:.1f} us -> 24 layers {24 * total / 1e3:.2f} ms")
