"""Network operator graphs on the tensorized operator set.

The paper evaluates its tensorized operators end to end on ResNet-50,
MobileNet-V2 and BERT-large; the reference kit itself has
no model import. Here a network is a flat list of `Op`s over named
fp16 NHWC activation buffers:

  conv    any tir_b200_conv geometry (C2D 3x3 / 7x7 / strided 1x1 ...) with the
          fused epilogue: bias (folded BatchNorm), fp16 residual, ReLU / ReLU6;
  gmm     a 1x1 stride-1 conv or a fully-connected layer as one GEMM over the
          zero-copy [pixels, C] view (TMA tiled operands), same epilogue;
  dep     depthwise 3x3 (MobileNet-V2) on the CUDA-core kernel, bias + ReLU6;
  maxpool / avgpool   the NHWC glue kernels (csrc/netops.cuh).

Every op is one C-ABI launch (two for CI=3 stems: the bit-exact (kw, c) relayout
plus the conv); the whole forward is captured once into a CUDA graph and
replayed. Batch sharding (shard.py): rank r of W builds the graph for its
samples [r*B/W, (r+1)*B/W) with replicated weights and no collective — the
shards are independent, so throughput scales with the number of GPUs.

Weights are random (He-normal, rounded to fp16; biases fp32): there is no
network access for checkpoints, and the benchmark metric does not depend on the
values. `oracle/nets_ref.py` replays the same op list in torch fp32 on the CPU
with the same fp16 rounding between layers (the parity reference).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import api


@dataclass
class Op:
    kind: str                       # conv | gmm | dep | maxpool | avgpool
    src: str
    dst: str
    spec: api.Conv | None = None    # conv / dep geometry (batch = the graph's batch)
    w: np.ndarray | None = None     # fp16 host weights: conv [K.., CI/G, CO], gmm [K, N], dep [KH, KW, C]
    b: np.ndarray | None = None     # fp32 host bias [CO]
    act: str = "none"               # none | relu | relu6
    res: str | None = None          # fp16 residual buffer (same shape as dst)
    pool: tuple = ()                # maxpool (k, s, p)
    out_f32: bool = False           # final logits


@dataclass
class NetDef:
    name: str
    batch: int
    input_shape: tuple              # (N, H, W, C)
    ops: list = field(default_factory=list)
    shapes: dict = field(default_factory=dict)   # buffer -> shape
    flops: int = 0                  # useful MAC*2 of the contractions (per forward)

    # -------------------------------------------------------------- builders
    def _new(self, shape):
        name = f"t{len(self.shapes)}"
        self.shapes[name] = tuple(shape)
        return name

    def conv(self, rng, x, co, k, s=1, p=0, act="relu", res=None, groups=1, w_scale=1.0):
        n, h, w, ci = self.shapes[x]
        dep = groups > 1 and groups == ci == co
        spec = api.Conv("DEP" if dep else "C2D", n=n, in_dhw=(1, h, w), ci=ci, co=co, k=(1, k, k),
                        s=(1, s, s), p=(0, p, p), groups=groups)
        oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        y = self._new((n, oh, ow, co))
        fan_in = k * k * (ci // groups)
        wshape = (k, k, co) if dep else (k, k, ci // groups, co)
        wt = (rng.standard_normal(wshape) * (w_scale * math.sqrt(2.0 / fan_in))).astype(np.float16)
        bias = (rng.standard_normal(co) * 0.01).astype(np.float32)
        self.flops += 2 * n * oh * ow * co * fan_in
        if k == 1 and s == 1 and p == 0 and groups == 1:
            self.ops.append(Op("gmm", x, y, w=wt.reshape(ci, co), b=bias, act=act, res=res))
        else:
            self.ops.append(Op("dep" if dep else "conv", x, y, spec=spec, w=wt, b=bias, act=act, res=res))
        return y

    def maxpool(self, x, k, s, p):
        n, h, w, c = self.shapes[x]
        y = self._new((n, (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1, c))
        self.ops.append(Op("maxpool", x, y, pool=(k, s, p)))
        return y

    def avgpool(self, x):
        n, h, w, c = self.shapes[x]
        y = self._new((n, 1, 1, c))
        self.ops.append(Op("avgpool", x, y))
        return y

    def fc(self, rng, x, classes):
        n, _, _, c = self.shapes[x]
        y = self._new((n, 1, 1, classes))
        wt = (rng.standard_normal((c, classes)) * math.sqrt(1.0 / c)).astype(np.float16)
        bias = (rng.standard_normal(classes) * 0.01).astype(np.float32)
        self.flops += 2 * n * c * classes
        self.ops.append(Op("gmm", x, y, w=wt, b=bias, act="none", out_f32=True))
        return y

    @property
    def output(self):
        return self.ops[-1].dst


def resnet50(batch: int, image: int = 224, classes: int = 1000, seed: int = 0) -> NetDef:
    """ResNet-50 v1.5 inference graph (BatchNorm folded into conv bias; stride on
    the 3x3 conv of each stage's first bottleneck; residual add + ReLU fused into
    the last 1x1 conv's epilogue)."""
    rng = np.random.default_rng(seed)
    net = NetDef("resnet50", batch, (batch, image, image, 3))
    x = net._new(net.input_shape)
    x = net.conv(rng, x, 64, 7, 2, 3)                    # stem (CI=3: (kw,c)-packed)
    x = net.maxpool(x, 3, 2, 1)
    for mid, blocks, stride in ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)):
        for i in range(blocks):
            s = stride if i == 0 else 1
            cout = mid * 4
            if i == 0:
                sc = net.conv(rng, x, cout, 1, s, 0, act="none")      # projection shortcut
            else:
                sc = x
            y = net.conv(rng, x, mid, 1, 1, 0)
            y = net.conv(rng, y, mid, 3, s, 1)
            x = net.conv(rng, y, cout, 1, 1, 0, act="relu", res=sc, w_scale=0.5)
    x = net.avgpool(x)
    net.fc(rng, x, classes)
    return net


def mobilenet_v2(batch: int, image: int = 224, classes: int = 1000, seed: int = 0) -> NetDef:
    """MobileNet-V2 (width 1.0) inference graph: expand 1x1 + ReLU6 -> DEP 3x3 +
    ReLU6 -> linear 1x1 projection (+ fused residual when shapes match)."""
    rng = np.random.default_rng(seed)
    net = NetDef("mobilenet_v2", batch, (batch, image, image, 3))
    x = net._new(net.input_shape)
    x = net.conv(rng, x, 32, 3, 2, 1, act="relu6")
    cin = 32
    for t, c, n, s in ((1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1),
                       (6, 160, 3, 2), (6, 320, 1, 1)):
        for i in range(n):
            stride = s if i == 0 else 1
            hidden = cin * t
            y = x if t == 1 else net.conv(rng, x, hidden, 1, act="relu6")
            y = net.conv(rng, y, hidden, 3, stride, 1, act="relu6", groups=hidden)
            res = x if (stride == 1 and cin == c) else None
            x = net.conv(rng, y, c, 1, act="none", res=res, w_scale=0.5 if res else 1.0)
            cin = c
    x = net.conv(rng, x, 1280, 1, act="relu6")
    x = net.avgpool(x)
    net.fc(rng, x, classes)
    return net


NETS = {"resnet50": resnet50, "mobilenet_v2": mobilenet_v2}


class DeviceNet:
    """A NetDef bound to one GPU: device weights, one buffer per activation, and
    the forward captured into a CUDA graph (`replay`)."""

    def __init__(self, net: NetDef, device):
        import torch

        self.net = net
        self.device = device
        self.buf = {k: torch.empty(v, dtype=torch.float16, device=device) for k, v in net.shapes.items()}
        out = net.output
        self.buf[out] = torch.empty(net.shapes[out], dtype=torch.float32, device=device)
        self.w, self.b = [], []
        for op in net.ops:
            self.w.append(torch.from_numpy(op.w).to(device) if op.w is not None else None)
            self.b.append(torch.from_numpy(op.b).to(device) if op.b is not None else None)
        self.graph = None
        self.stream = torch.cuda.Stream(device=device)

    @property
    def input(self):
        return self.buf[self.net.ops[0].src]

    @property
    def output(self):
        return self.buf[self.net.output]

    def run(self, lo: int = 0, hi: int | None = None):
        """Eager forward (ops [lo, hi)) on self.stream: one C-ABI call per op."""
        ops = self.net.ops
        for i in range(lo, len(ops) if hi is None else hi):
            op = ops[i]
            x, y = self.buf[op.src], self.buf[op.dst]
            res = self.buf[op.res] if op.res else None
            if op.kind in ("conv", "dep"):
                api.conv(op.spec, x, self.w[i], y, out_f16=True, bias=self.b[i], relu=op.act,
                         residual=res, stream=self.stream)
            elif op.kind == "gmm":
                k, n = op.w.shape
                a = x.view(-1, k)
                c = y.view(-1, n)
                r = res.view(-1, n) if res is not None else None
                api.gmm(a, self.w[i], c, out_f16=not op.out_f32, bias=self.b[i], relu=op.act, residual=r,
                        stream=self.stream)
            elif op.kind == "maxpool":
                api.maxpool2d(x, *op.pool, Y=y, stream=self.stream)
            elif op.kind == "avgpool":
                api.avgpool_global(x, Y=y.view(y.shape[0], y.shape[3]), stream=self.stream)
            else:
                raise api.TirError("ValueError", f"unknown op kind {op.kind}")

    def capture(self):
        """Warm up (sizes the library workspace) and capture the forward."""
        import torch

        with torch.cuda.stream(self.stream):
            self.run()
        self.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        api.reset_launch_count()
        with torch.cuda.graph(g, stream=self.stream, capture_error_mode="relaxed"):
            self.run()
        self.launches = api.launch_count()  # kernels in one captured forward (library counter)
        self.graph = g
        return g

    def replay(self):
        """One forward: graph replay on self.stream (graphs launch on the current stream)."""
        import torch

        with torch.cuda.stream(self.stream):
            self.graph.replay()


def launches_per_forward(net) -> int:
    """Kernel launches of one forward (CI % 8 != 0 stems add the two relayout kernels;
    a BERT layer is 9 launches)."""
    if isinstance(net, BertDef):
        return 9 * net.layers
    n = 0
    for op in net.ops:
        n += 1
        if op.kind == "conv" and op.spec.ci % 8:
            n += 2
    return n


def build_shard(name: str, global_batch: int, rank: int, world: int, **kw):
    """(net definition of this rank's samples, (lo, hi)) — same seed, so weights are replicated."""
    from . import shard

    lo, hi = shard.batch_range(global_batch, rank, world)
    return NETS[name](hi - lo, **kw), (lo, hi)


# ---------------------------------------------------------------------- BERT

@dataclass
class BertDef:
    """BERT encoder stack (post-LN, GELU FFN) on fp16 hidden states [B*S, H]:
    per layer QKV GEMM (+bias) -> batched Q K^T over (sequence, head), K read
    in place from QKV as a K-major operand -> softmax(scale) -> batched P V -> output GEMM (+bias +residual) ->
    LayerNorm -> FFN GEMM (+bias, GELU) -> GEMM (+bias +residual) -> LayerNorm.
    The token embedding lookup is not part of the operator graph: the input is
    the embedded hidden-state tensor."""

    name: str
    batch: int
    seq: int = 512
    hidden: int = 1024
    heads: int = 16
    ffn: int = 4096
    layers: int = 24
    eps: float = 1e-12
    weights: list = field(default_factory=list)  # per layer dict of host arrays

    @property
    def tokens(self):
        return self.batch * self.seq

    @property
    def head_dim(self):
        return self.hidden // self.heads

    @property
    def input_shape(self):
        return (self.tokens, self.hidden)

    @property
    def flops(self):
        t, h, f, s = self.tokens, self.hidden, self.ffn, self.seq
        dense = 2 * t * (3 * h * h + h * h + 2 * h * f)
        attn = 2 * 2 * self.batch * self.heads * s * s * self.head_dim
        return self.layers * (dense + attn)


def bert_large(batch: int, seq: int = 512, layers: int = 24, hidden: int = 1024, heads: int = 16,
               ffn: int = 4096, seed: int = 0) -> BertDef:
    rng = np.random.default_rng(seed)
    net = BertDef("bert_large", batch, seq, hidden, heads, ffn, layers)
    for _ in range(layers):
        w = {}
        for key, (k, n) in (("qkv", (hidden, 3 * hidden)), ("o", (hidden, hidden)), ("f1", (hidden, ffn)),
                            ("f2", (ffn, hidden))):
            w["w_" + key] = (rng.standard_normal((k, n)) * (0.5 / math.sqrt(k))).astype(np.float16)
            w["b_" + key] = (rng.standard_normal(n) * 0.02).astype(np.float32)
        for ln in ("ln1", "ln2"):
            w[ln + "_g"] = (1.0 + 0.1 * rng.standard_normal(hidden)).astype(np.float32)
            w[ln + "_b"] = (0.1 * rng.standard_normal(hidden)).astype(np.float32)
        net.weights.append(w)
    return net


NETS["bert_large"] = bert_large


class DeviceBert:
    """BertDef on one GPU: device weights, shared activation buffers, CUDA-graph forward."""

    def __init__(self, net: BertDef, device):
        import torch

        self.net = net
        self.device = device
        t, h, f = net.tokens, net.hidden, net.ffn
        e = lambda *s: torch.empty(s, dtype=torch.float16, device=device)  # noqa: E731
        self.x = e(t, h)          # layer input / output (hidden states)
        self.qkv = e(t, 3 * h)
        self.scores = e(net.batch * net.heads * net.seq, net.seq)
        self.ctx = e(t, h)
        self.attn = e(t, h)
        self.x1 = e(t, h)
        self.hid = e(t, f)
        self.y = e(t, h)
        self.w = [{k: torch.from_numpy(v).to(device) for k, v in lw.items()} for lw in net.weights]
        self.stream = torch.cuda.Stream(device=device)
        self.graph = None

    @property
    def input(self):
        return self.x

    @property
    def output(self):
        return self.x

    def run(self, lo: int = 0, hi: int | None = None):
        net, st = self.net, self.stream
        B, S, H, nh, dh = net.batch, net.seq, net.hidden, net.heads, net.head_dim
        for li in range(lo, net.layers if hi is None else hi):
            w = self.w[li]
            api.gmm(self.x, w["w_qkv"], self.qkv, out_f16=True, bias=w["b_qkv"], stream=st)
            # scores[(b*nh + h)*S + m, n] = Q[b*S + m, h*dh + k] . K[b*S + n, H + h*dh + k]
            # (K read straight from QKV as a K-major B operand: no transpose)
            api.gmm_batched(self.qkv, self.qkv, self.scores, S, S, dh, (B, nh),
                            a=((0, S, 0), (0, 0, dh)), b=((0, S, 0), (H, 0, dh)),
                            c=((0, nh * S, S), (0, 0, 0)), b_kmajor=True, stream=st)
            api.softmax(self.scores, 1.0 / math.sqrt(dh), Y=self.scores, stream=st)
            # ctx[b*S + m, h*dh + n] = P[(b*nh + h)*S + m, k] . V[b*S + k, 2H + h*dh + n]
            api.gmm_batched(self.scores, self.qkv, self.ctx, S, dh, S, (B, nh),
                            a=((0, nh * S, S), (0, 0, 0)), b=((0, S, 0), (2 * H, 0, dh)),
                            c=((0, S, 0), (0, 0, dh)), stream=st)
            api.gmm(self.ctx, w["w_o"], self.attn, out_f16=True, bias=w["b_o"], residual=self.x, stream=st)
            api.layernorm(self.attn, w["ln1_g"], w["ln1_b"], net.eps, Y=self.x1, stream=st)
            api.gmm(self.x1, w["w_f1"], self.hid, out_f16=True, bias=w["b_f1"], relu="gelu", stream=st)
            api.gmm(self.hid, w["w_f2"], self.y, out_f16=True, bias=w["b_f2"], residual=self.x1, stream=st)
            api.layernorm(self.y, w["ln2_g"], w["ln2_b"], net.eps, Y=self.x, stream=st)

    def capture(self):
        import torch

        with torch.cuda.stream(self.stream):
            self.run()
        self.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        api.reset_launch_count()
        with torch.cuda.graph(g, stream=self.stream, capture_error_mode="relaxed"):
            self.run()
        self.launches = api.launch_count()  # kernels in one captured forward (library counter)
        self.graph = g
        return g

    def replay(self):
        import torch

        with torch.cuda.stream(self.stream):
            self.graph.replay()


def device_net(net, device):
    """DeviceNet for conv graphs, DeviceBert for BERT."""
    return DeviceBert(net, device) if isinstance(net, BertDef) else DeviceNet(net, device)
