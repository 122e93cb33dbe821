"""One small launch of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): igemm_tc_kernel (tiled GMM, im2col conv,
T2D sub-pixel classes, cta_group::2 pairs, cluster split-K with the fused
epilogue, batched attention GEMM), conv_halo_kernel, dep_tile_kernel and the
untiled dep_kernel, conv_rowpack_kernel (C3D / DIL / fused stem), the relayout kernels (channel pad, (kw, c) and
(kh, kw, c) packing), and the network glue (pooling, LayerNorm, softmax).
Each result is checked so a sanitizer run also proves the launches computed.

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)


def rnd(*s):
    return torch.randn(*s, device=dev, generator=g).half()


def ref_conv(spec, x, w):
    import torch.nn.functional as F

    r = spec.spatial_rank
    xt = x.double().movedim(-1, 1)
    if spec.op == "DEP":
        wt = w.double().movedim(-1, 0).unsqueeze(1)
    else:
        wt = w.double().movedim(-1, 0).movedim(-1, 1)
    k = dict(stride=spec.s[3 - r:], padding=spec.p[3 - r:], dilation=spec.d[3 - r:], groups=spec.groups)
    y = [F.conv1d, F.conv2d, F.conv3d][r - 1](xt, wt, **k)
    return y.movedim(1, -1)


def check(name, got, want, tol=2e-2):
    err = (got.double() - want).abs().max().item() / max(want.abs().max().item(), 1e-6)
    print(f"{name}: rel err {err:.2e}", flush=True)
    assert err < tol, name


cases = {
    "C2D halo": tb.Conv("C2D", n=1, in_dhw=(1, 9, 9), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1)),
    "C2D im2col s2": tb.Conv("C2D", n=1, in_dhw=(1, 9, 9), ci=64, co=64, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1)),
    "C1D": tb.Conv("C1D", n=2, in_dhw=(1, 1, 33), ci=64, co=64, k=(1, 1, 3), s=(1, 1, 2), p=(0, 0, 1)),
    "C3D ci3": tb.Conv("C3D", n=1, in_dhw=(4, 8, 8), ci=3, co=32, k=(3, 3, 3), s=(2, 2, 2), p=(1, 1, 1)),
    "DIL ci3": tb.Conv("DIL", n=1, in_dhw=(1, 16, 16), ci=3, co=32, k=(1, 3, 3), p=(0, 2, 2), d=(1, 2, 2)),
    "GRP": tb.Conv("GRP", n=1, in_dhw=(1, 8, 8), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1), groups=2),
    "DEP tile": tb.Conv("DEP", n=1, in_dhw=(1, 16, 32), ci=32, co=32, k=(1, 3, 3), p=(0, 1, 1), groups=32),
    "DEP simple": tb.Conv("DEP", n=1, in_dhw=(1, 7, 7), ci=12, co=12, k=(1, 5, 5), p=(0, 2, 2), groups=12),
    # conv_rowpack_kernel: A operand packed in TMEM (7x7x3 window; w-dilated window; 3-D depth ring)
    "C3D rowpack 7^3": tb.Conv("C3D", n=1, in_dhw=(7, 16, 24), ci=3, co=64, k=(7, 7, 7), s=(2, 2, 2), p=(3, 3, 3)),
    "DIL rowpack d2": tb.Conv("DIL", n=1, in_dhw=(1, 24, 40), ci=3, co=64, k=(1, 7, 7), s=(1, 2, 2), p=(0, 3, 3),
                              d=(1, 2, 2)),
}
for name, spec in cases.items():
    x, w = rnd(*spec.x_shape()), rnd(*spec.w_shape())
    check(name, tb.conv(spec, x, w), ref_conv(spec, x, w))
spec = tb.Conv("C2D", n=2, in_dhw=(1, 24, 40), ci=3, co=32, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1))
x, w = rnd(*spec.x_shape()), rnd(*spec.w_shape())
bias = torch.randn(32, device=dev, generator=g)
check("stem rowpack + bias/ReLU6 fp16", tb.conv(spec, x, w, bias=bias, relu="relu6", out_f16=True),
      ref_conv(spec, x, w).add(bias.double()).clamp(0, 6))
spec = tb.Conv("T2D", n=1, in_dhw=(1, 4, 4), ci=64, co=64, k=(1, 4, 4), s=(1, 2, 2), p=(0, 1, 1), transposed=True)
x, w = rnd(*spec.x_shape()), rnd(*spec.w_shape())
y = tb.conv(spec, x, w)
torch.cuda.synchronize()
print("T2D: finite", bool(torch.isfinite(y).all()), flush=True)

a, b = rnd(256, 128), rnd(128, 256)
check("GMM pairs (cta_group::2)", tb.gmm(a, b), a.double() @ b.double())
tb.set_option("ksplit", 2)
bias = torch.randn(256, device=dev, generator=g)
res = rnd(256, 256)
check("GMM cluster split-K + epilogue", tb.gmm(a, b, out_f16=True, bias=bias, relu=True, residual=res),
      torch.relu(a.double() @ b.double() + bias.double() + res.double()))
tb.set_option("ksplit", 0)
q = rnd(256, 64)
c = torch.zeros(256, 256, device=dev).half()
tb.gmm_batched(q, q, c, 128, 128, 64, (2, 1), a=((0, 128, 0), (0, 0, 0)), b=((0, 128, 0), (0, 0, 0)),
               c=((0, 128, 0), (0, 128, 0)), b_kmajor=True)
check("batched K-major", c[:128, :128], q[:128].double() @ q[:128].double().t())

x = rnd(2, 8, 8, 32)
check("maxpool", tb.maxpool2d(x, 3, 2, 1), torch.nn.functional.max_pool2d(
    x.double().movedim(-1, 1), 3, 2, 1).movedim(1, -1), 1e-3)
check("avgpool", tb.avgpool_global(x), x.double().mean(dim=(1, 2)), 1e-2)
h = rnd(64, 256)
gm, bt = torch.randn(256, device=dev, generator=g), torch.randn(256, device=dev, generator=g)
check("layernorm", tb.layernorm(h, gm, bt, 1e-5), torch.nn.functional.layer_norm(
    h.double(), (256,), gm.double(), bt.double(), 1e-5))
check("softmax", tb.softmax(h, 0.125), torch.softmax(h.double() * 0.125, -1))
torch.cuda.synchronize()
print("SANITIZE_CASES_OK", flush=True)
