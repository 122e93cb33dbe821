"""CPU reference of the network graphs — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Replays a `paper_2207_04296_b200.nets.NetDef` op list with torch on the CPU in
float64, rounding every fp16 activation exactly where the device graph stores
fp16 (conv / gmm / pool outputs), so the only differences left are the fp32
accumulation order inside the tensor cores (about K * 2^-24 relative) and the
fp16 rounding flips it occasionally causes. Used by tests/test_gpu_nets.py and
the gloo sharding test; the networks have no counterpart in /root/reference
(the kit has no model import), so this restates torch's conv2d /
max_pool2d / mean semantics, per layer, in the NHWC / HWIO conventions of
include/tir_b200.h.
"""
from __future__ import annotations

import numpy as np


def _act(t, act):
    import torch

    if act == "relu":
        return torch.clamp_min(t, 0.0)
    if act == "relu6":
        return torch.clamp(t, 0.0, 6.0)
    if act == "gelu":
        return torch.nn.functional.gelu(t)
    return t


def _f16(t):
    import torch

    return t.to(torch.float16).to(torch.float64)


def forward(net, x: np.ndarray) -> np.ndarray:
    """Logits [N, classes] (float64) of `net` on fp16 NHWC input `x`."""
    import torch
    import torch.nn.functional as F

    bufs = {net.ops[0].src: torch.from_numpy(np.asarray(x, np.float16)).to(torch.float64)}
    for op in net.ops:
        xin = bufs[op.src]
        if op.kind in ("conv", "dep"):
            sp = op.spec
            xn = xin.permute(0, 3, 1, 2)
            w = torch.from_numpy(op.w).to(torch.float64)
            if op.kind == "dep":
                wt = w.permute(2, 0, 1).unsqueeze(1)          # [C, 1, KH, KW]
            else:
                wt = w.permute(3, 2, 0, 1)                    # [CO, CI/G, KH, KW]
            y = F.conv2d(xn, wt, stride=sp.s[1:], padding=sp.p[1:], dilation=sp.d[1:], groups=sp.groups)
            y = y.permute(0, 2, 3, 1)
        elif op.kind == "gmm":
            k, n = op.w.shape
            y = (xin.reshape(-1, k) @ torch.from_numpy(op.w).to(torch.float64))
            y = y.reshape(*xin.shape[:-1], n)
        elif op.kind == "maxpool":
            k, s, p = op.pool
            y = F.max_pool2d(xin.permute(0, 3, 1, 2), k, s, p).permute(0, 2, 3, 1)
        elif op.kind == "avgpool":
            y = xin.mean(dim=(1, 2), keepdim=True)
        else:
            raise ValueError(op.kind)
        if op.b is not None:
            y = y + torch.from_numpy(op.b).to(torch.float64)
        if op.res is not None:
            y = y + bufs[op.res]
        y = _act(y, op.act)
        bufs[op.dst] = y if op.out_f32 else _f16(y)
    out = bufs[net.output]
    return out.reshape(out.shape[0], -1).numpy()


def bert_forward(net, x: np.ndarray) -> np.ndarray:
    """Hidden states after `net.layers` encoder layers (float64, with the device
    graph's fp16 rounding points: QKV, K^T (exact), scores, probabilities,
    context, every GEMM output and both LayerNorms)."""
    import torch

    f16 = _f16
    t = lambda a: torch.from_numpy(a).to(torch.float64)  # noqa: E731
    B, S, H, nh, dh = net.batch, net.seq, net.hidden, net.heads, net.head_dim
    xh = t(np.asarray(x, np.float16))
    for w in net.weights:
        qkv = f16(xh @ t(w["w_qkv"]) + t(w["b_qkv"]))
        q = qkv[:, :H].reshape(B, S, nh, dh).permute(0, 2, 1, 3)
        k = qkv[:, H:2 * H].reshape(B, S, nh, dh).permute(0, 2, 1, 3)
        v = qkv[:, 2 * H:].reshape(B, S, nh, dh).permute(0, 2, 1, 3)
        scores = f16(q @ k.transpose(-1, -2))
        p = f16(torch.softmax(scores / np.sqrt(dh), dim=-1))
        ctx = f16((p @ v).permute(0, 2, 1, 3).reshape(B * S, H))
        attn = f16(ctx @ t(w["w_o"]) + t(w["b_o"]) + xh)
        x1 = f16(torch.nn.functional.layer_norm(attn, (H,), t(w["ln1_g"]), t(w["ln1_b"]), net.eps))
        hid = f16(torch.nn.functional.gelu(x1 @ t(w["w_f1"]) + t(w["b_f1"])))
        y = f16(hid @ t(w["w_f2"]) + t(w["b_f2"]) + x1)
        xh = f16(torch.nn.functional.layer_norm(y, (H,), t(w["ln2_g"]), t(w["ln2_b"]), net.eps))
    return xh.numpy()
