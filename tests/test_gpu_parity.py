"""GPU parity: every CUDA kernel against the oracle, through the C-ABI.

Bars:
  * D1 — the reference's input distribution (workloads.h:170-184): every
    partial sum is exact in fp32, so results must be BIT-EXACT (value equality
    as the reference's tensors_bitwise_equal defines it, workloads.h:284-298);
  * D2 — N(0,1) rounded to fp16: every element within rel 1e-4 under
    tensors_close (workloads.h:264-282) OR within 1e-6 (~16 fp32 ulp) of its
    dot product's absolute sum sum|a*b| (oracle.tensors_close_dot: tensor cores
    reassociate the fp32 sum, which is only accurate relative to sum|a*b| when
    the result cancels); DEP (no-FMA, reference order) is bit-exact on D2 too;
  * paper shapes: exact on D1 for sampled images (outputs are independent per
    image), plus size-independent properties on the full output (linearity in
    the weights, accumulate == out + Yin, fp16 output == RN(fp32 output)).
"""
import numpy as np
import pytest

import paper_2207_04296_b200 as tb
from oracle import ir_gen as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu

REL_TOL_D2 = 1e-4
DOT_TOL_D2 = 1e-6


def ospec(spec: tb.Conv) -> G.ConvSpec:
    return G.ConvSpec(op=spec.op, n=spec.n, in_dhw=spec.in_dhw, ci=spec.ci, co=spec.co, k=spec.k,
                      s=spec.s, p=spec.p, d=spec.d, groups=spec.groups, transposed=spec.transposed)


def dev(x, cuda):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(cuda).half()


def run_conv(spec, x, w, cuda, **kw):
    import torch

    y = tb.conv(spec, dev(x, cuda), dev(w, cuda), **kw)
    torch.cuda.synchronize()
    return y.float().cpu().numpy()


SMALL = {
    "C1D": tb.Conv("C1D", n=3, in_dhw=(1, 1, 37), ci=64, co=128, k=(1, 1, 3), s=(1, 1, 2), p=(0, 0, 1)),
    "C2D": tb.Conv("C2D", n=2, in_dhw=(1, 11, 13), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1)),
    "C2D_s2_ci128": tb.Conv("C2D", n=2, in_dhw=(1, 15, 15), ci=128, co=64, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1)),
    "C2D_1x1": tb.Conv("C2D", n=1, in_dhw=(1, 9, 9), ci=64, co=256, k=(1, 1, 1)),
    "C2D_ci32": tb.Conv("C2D", n=2, in_dhw=(1, 9, 9), ci=32, co=64, k=(1, 3, 3), p=(0, 1, 1)),
    "C2D_ci16": tb.Conv("C2D", n=2, in_dhw=(1, 9, 9), ci=16, co=32, k=(1, 3, 3), p=(0, 1, 1)),
    "C2D_ci8": tb.Conv("C2D", n=2, in_dhw=(1, 9, 9), ci=8, co=16, k=(1, 3, 3), p=(0, 1, 1)),
    "C2D_ci96_co40": tb.Conv("C2D", n=1, in_dhw=(1, 7, 10), ci=96, co=40, k=(1, 3, 5), p=(0, 1, 2)),
    "C3D": tb.Conv("C3D", n=1, in_dhw=(6, 12, 12), ci=3, co=64, k=(7, 7, 7), s=(2, 2, 2), p=(3, 3, 3)),
    "C3D_ci16": tb.Conv("C3D", n=2, in_dhw=(4, 6, 6), ci=16, co=32, k=(3, 3, 3), p=(1, 1, 1)),
    # rowpack kernel (A operand packed in TMEM, rowpack.cuh): partial tiles in h and w, two depth groups
    "C3D_rp": tb.Conv("C3D", n=2, in_dhw=(7, 24, 40), ci=3, co=64, k=(7, 7, 7), s=(2, 2, 2), p=(3, 3, 3)),
    # CO = 32 (SW64 weight panel) and an odd output depth count (a one-depth group)
    "C3D_rp_odd": tb.Conv("C3D", n=1, in_dhw=(5, 16, 16), ci=3, co=32, k=(7, 7, 7), s=(2, 2, 2), p=(3, 3, 3)),
    # 2-D stems: ResNet-50's 7x7 s2 and MobileNet-V2's 3x3 s2 (CI = 3)
    "C2D_stem7": tb.Conv("C2D", n=2, in_dhw=(1, 32, 32), ci=3, co=64, k=(1, 7, 7), s=(1, 2, 2), p=(0, 3, 3)),
    "C2D_stem3": tb.Conv("C2D", n=2, in_dhw=(1, 24, 40), ci=3, co=32, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1)),
    # rowpack with a dilated (kw, c) window (the DIL paper geometry on a small image)
    "DIL_rp": tb.Conv("DIL", n=2, in_dhw=(1, 40, 48), ci=3, co=64, k=(1, 7, 7), s=(1, 2, 2), p=(0, 3, 3), d=(1, 2, 2)),
    "DIL": tb.Conv("DIL", n=1, in_dhw=(1, 30, 30), ci=3, co=64, k=(1, 7, 7), s=(1, 2, 2), p=(0, 3, 3), d=(1, 2, 2)),
    "DIL_ci64": tb.Conv("DIL", n=2, in_dhw=(1, 14, 14), ci=64, co=64, k=(1, 3, 3), p=(0, 2, 2), d=(1, 2, 2)),
    "GRP": tb.Conv("GRP", n=2, in_dhw=(1, 12, 12), ci=64, co=128, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=4),
    "GRP_g2": tb.Conv("GRP", n=1, in_dhw=(1, 10, 10), ci=128, co=128, k=(1, 3, 3), p=(0, 1, 1), groups=2),
    # group-packed igemm (GP): 4 groups of 16 channels per 64-channel piece, two piece blocks (G = 8)
    "GRP_gp16": tb.Conv("GRP", n=2, in_dhw=(1, 13, 11), ci=128, co=256, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1),
                        groups=8),
    # GP with 2 groups of 32 channels per piece (BN = 64), a 1x7 window (taps * cig <= 256)
    "GRP_gp32": tb.Conv("GRP", n=1, in_dhw=(1, 9, 12), ci=64, co=64, k=(1, 1, 7), p=(0, 0, 3), groups=2),
    # rowpack: an image narrower than one 16-column tile (Wt = OW) and a 3-D shape with depth stride 1
    "C2D_stem7_narrow": tb.Conv("C2D", n=3, in_dhw=(1, 20, 16), ci=3, co=64, k=(1, 7, 7), s=(1, 2, 2), p=(0, 3, 3)),
    "C3D_rp_s1d": tb.Conv("C3D", n=1, in_dhw=(5, 16, 16), ci=3, co=32, k=(3, 3, 3), s=(1, 2, 2), p=(1, 1, 1)),
    "T2D": tb.Conv("T2D", n=2, in_dhw=(1, 4, 4), ci=64, co=64, k=(1, 4, 4), s=(1, 2, 2), p=(0, 1, 1), transposed=True),
    "T2D_k3": tb.Conv("T2D", n=1, in_dhw=(1, 5, 6), ci=64, co=32, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), transposed=True),
    "DEP": tb.Conv("DEP", n=2, in_dhw=(1, 9, 9), ci=32, co=32, k=(1, 3, 3), p=(0, 1, 1), groups=32),
    "DEP_s2": tb.Conv("DEP", n=2, in_dhw=(1, 28, 28), ci=96, co=96, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=96),
    # more tiles than resident blocks: exercises the second TMA ring slot (128-B aligned)
    "DEP_s2_ring": tb.Conv("DEP", n=8, in_dhw=(1, 112, 112), ci=96, co=96, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1),
                           groups=96),
    # narrow-image tile variants (MobileNet-V2 14x14 / 7x7 stages)
    "DEP_14": tb.Conv("DEP", n=3, in_dhw=(1, 14, 14), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1), groups=64),
    "DEP_7": tb.Conv("DEP", n=5, in_dhw=(1, 7, 7), ci=96, co=96, k=(1, 3, 3), p=(0, 1, 1), groups=96),
    "DEP_s2_14": tb.Conv("DEP", n=3, in_dhw=(1, 14, 14), ci=64, co=64, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1),
                         groups=64),
    # C % 32 != 0: partial last channel block in the TMA tile kernel (MobileNet-V2 144 / 24 channels)
    "DEP_c144": tb.Conv("DEP", n=2, in_dhw=(1, 20, 20), ci=144, co=144, k=(1, 3, 3), p=(0, 1, 1), groups=144),
    "DEP_c40_s2": tb.Conv("DEP", n=2, in_dhw=(1, 17, 17), ci=40, co=40, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1),
                          groups=40),
    "DEP_c12": tb.Conv("DEP", n=1, in_dhw=(1, 7, 7), ci=12, co=12, k=(1, 5, 5), p=(0, 2, 2), groups=12),
    # tile shape by width (tir_b200.cu dep_impl): 112 wide takes 16 x 16 tiles; 14 wide with
    # more 8 x 8 tiles than two waves of CTAs (16 x 2 x 2 x 18 > 888) takes 16 x 16 too
    "DEP_w112": tb.Conv("DEP", n=2, in_dhw=(1, 112, 112), ci=32, co=32, k=(1, 3, 3), p=(0, 1, 1), groups=32),
    "DEP_w14_many": tb.Conv("DEP", n=16, in_dhw=(1, 14, 14), ci=576, co=576, k=(1, 3, 3), p=(0, 1, 1),
                            groups=576),
}


@pytest.mark.parametrize("name", list(SMALL))
def test_conv_d1_bit_exact(name, cuda):
    spec = SMALL[name]
    x = O.reference_tensor(spec.x_shape(), 1)
    w = O.reference_tensor(spec.w_shape(), 2)
    got = run_conv(spec, x, w, cuda)
    want = O.conv(ospec(spec), x, w, threads=8)
    assert O.tensors_bitwise_equal(got, want), f"max diff {np.abs(got - want).max()}"


@pytest.mark.parametrize("name", list(SMALL))
def test_conv_d2_within_tolerance(name, cuda):
    spec = SMALL[name]
    x = O.normal_f16(spec.x_shape(), 3)
    w = O.normal_f16(spec.w_shape(), 4)
    got = run_conv(spec, x, w, cuda)
    want = O.conv(ospec(spec), x, w, threads=8)
    abs_sum = O.conv(ospec(spec), np.abs(x), np.abs(w), threads=8)
    assert O.tensors_close_dot(got, want, abs_sum, REL_TOL_D2, DOT_TOL_D2)
    if spec.op == "DEP":  # reference-ordered, no-FMA accumulation
        assert O.tensors_bitwise_equal(got, want)


@pytest.mark.parametrize("name", ["C2D", "GRP", "T2D", "DEP", "C1D", "C3D_rp", "C2D_stem3", "DIL_rp", "GRP_gp16",
                                  "GRP_gp32"])
def test_conv_accumulate_and_fp16_out(name, cuda):
    import torch

    spec = SMALL[name]
    x = O.reference_tensor(spec.x_shape(), 5)
    w = O.reference_tensor(spec.w_shape(), 6)
    y0 = O.reference_tensor(spec.y_shape(), 7)
    Y = torch.from_numpy(y0.copy()).to(cuda)
    tb.conv(spec, dev(x, cuda), dev(w, cuda), Y, accumulate=True)
    torch.cuda.synchronize()
    want = O.conv(ospec(spec), x, w, y0, threads=8)
    assert O.tensors_bitwise_equal(Y.cpu().numpy(), want)
    yh = run_conv(spec, x, w, cuda, out_f16=True)
    ref = O.conv(ospec(spec), x, w, threads=8).astype(np.float16).astype(np.float32)
    assert np.array_equal(yh, ref)


@pytest.mark.parametrize("op", ["C1D", "C2D", "GRP", "T2D", "DEP", "DIL"])
def test_paper_shape_sampled_images_exact(op, cuda):
    spec = tb.PAPER_SHAPES[op]
    x = O.reference_tensor(spec.x_shape(), 11)
    w = O.reference_tensor(spec.w_shape(), 12)
    got = run_conv(spec, x, w, cuda)
    one = ospec(spec.with_(n=1))
    for img in (0, spec.n - 1):
        want = O.conv(one, x[img:img + 1], w, threads=8)
        assert O.tensors_bitwise_equal(got[img:img + 1], want), f"image {img}"


def test_paper_c3d_sampled_rows_exact(cuda):
    # C3D is 1.06e11 MACs: check output slices of the first image (an output
    # row only depends on its own receptive field, so a cropped problem with
    # the same geometry reproduces it exactly).
    spec = tb.PAPER_SHAPES["C3D"]
    x = O.reference_tensor(spec.x_shape(), 13)
    w = O.reference_tensor(spec.w_shape(), 14)
    got = run_conv(spec, x, w, cuda)
    assert np.isfinite(got).all()
    # depth slices 0..1 of image 0: inputs d in [0, 2*1+7-3) -> crop depth 6
    crop = spec.with_(n=1, in_dhw=(6, 224, 224))
    want = O.conv(ospec(crop), x[:1, :6], w, threads=16)
    assert O.tensors_bitwise_equal(got[:1, :2], want[:, :2])


def test_paper_c2d_properties_full_size(cuda):
    import torch

    spec = tb.PAPER_SHAPES["C2D"]
    X = torch.randn(*spec.x_shape(), device=cuda).half()
    W1 = torch.randn(*spec.w_shape(), device=cuda).half()
    W2 = torch.randn(*spec.w_shape(), device=cuda).half()
    y1 = tb.conv(spec, X, W1)
    y2 = tb.conv(spec, X, W2)
    # linearity in the weights: doubling W is exact in fp16 and fp32, so Y doubles exactly
    y2x = tb.conv(spec, X, (W1.float() * 2).half())
    assert torch.equal(y2x, y1 * 2)
    # accumulate == previous + fresh
    acc = y1.clone()
    tb.conv(spec, X, W2, acc, accumulate=True)
    torch.testing.assert_close(acc, y1 + y2, rtol=1e-5, atol=1e-4)
    # fp16 output is RN of the fp32 output
    yh = tb.conv(spec, X, W1, out_f16=True)
    assert torch.equal(yh, y1.half())


GMM_CASES = [(128, 64, 64), (256, 128, 256), (200, 64, 128), (128, 64, 72), (256, 48, 128),
             (1, 16, 16), (129, 8, 8), (1024, 1024, 1024), (333, 520, 264)]


@pytest.mark.parametrize("mnk", GMM_CASES, ids=lambda t: "x".join(map(str, t)))
def test_gmm_d1_bit_exact(mnk, cuda):
    import torch

    M, N, K = mnk
    a = O.reference_tensor((M, K), 1)
    b = O.reference_tensor((K, N), 2)
    c = tb.gmm(dev(a, cuda), dev(b, cuda))
    torch.cuda.synchronize()
    rows = min(M, 128)
    assert O.tensors_bitwise_equal(c.cpu().numpy()[:rows], O.gmm(a[:rows], b, threads=8))
    assert O.tensors_bitwise_equal(c.cpu().numpy()[-rows:], O.gmm(a[-rows:], b, threads=8))


@pytest.mark.parametrize("mnk", [(256, 128, 512), (333, 520, 264)], ids=lambda t: "x".join(map(str, t)))
def test_gmm_d2_and_variants(mnk, cuda):
    import torch

    M, N, K = mnk
    a = O.normal_f16((M, K), 3)
    b = O.normal_f16((K, N), 4)
    c0 = O.normal_f16((M, N), 5)
    want = O.gmm(a, b, threads=8)
    c = tb.gmm(dev(a, cuda), dev(b, cuda))
    C = torch.from_numpy(c0.copy()).to(cuda)
    tb.gmm(dev(a, cuda), dev(b, cuda), C, accumulate=True)
    ch = tb.gmm(dev(a, cuda), dev(b, cuda), out_f16=True)
    torch.cuda.synchronize()
    abs_sum = O.gmm(np.abs(a), np.abs(b), threads=8)
    assert O.tensors_close_dot(c.cpu().numpy(), want, abs_sum, REL_TOL_D2, DOT_TOL_D2)
    assert O.tensors_close_dot(C.cpu().numpy(), O.gmm(a, b, c0, threads=8), abs_sum + np.abs(c0),
                               REL_TOL_D2, DOT_TOL_D2)
    # fp16 output = RN of an fp32 sum; the fp32-output launch may split K (a
    # different fp32 summation order), so on N(0,1) data the two agree to one fp16 ulp
    c32 = c.cpu().numpy()
    c16 = c32.astype(np.float16)
    got16 = ch.cpu().numpy()
    ulp = np.spacing(np.abs(c16)).astype(np.float32)
    # one fp16 ulp, plus the reassociation bound of the two fp32 sums where the result cancels
    assert (np.abs(got16.astype(np.float32) - c16.astype(np.float32)) <= ulp + 2 * DOT_TOL_D2 * abs_sum).all()
    assert np.mean(got16 == c16) > 0.99


@pytest.mark.parametrize("mnk", [(1024, 1024, 1024), (2048, 512, 2048), (384, 256, 256), (4096, 1024, 4096)],
                         ids=lambda t: "x".join(map(str, t)))
def test_gmm_cta_pairs(mnk, option, cuda):
    """CTA-pair GEMMs (igemm.cuh mc_tile): the default tcgen05.mma.cta_group::2 pairs
    (M = 256, half of B per SM) give bit-identical results to unpaired launches
    (option mc = 0) — the same K order per output — plain and with the fused bias /
    GELU / residual fp16 epilogue, and are bit-exact vs the oracle on the reference
    distribution. 384 rows = 3 M tiles (odd) falls back to unpaired launches."""
    import torch

    M, N, K = mnk
    a = O.reference_tensor((M, K), 1)
    b = O.reference_tensor((K, N), 2)
    an, bn_ = O.normal_f16((M, K), 3), O.normal_f16((K, N), 4)
    bias = torch.randn(N, device=cuda)
    res = torch.randn(M, N, device=cuda).half()
    outs = {}
    for mode, mc in (("unpaired", 0), ("cta_group2", 1)):
        option("mc", mc)
        acc = torch.from_numpy(O.normal_f16((M, N), 5).astype(np.float32)).to(cuda)
        tb.gmm(dev(an, cuda), dev(bn_, cuda), acc, accumulate=True)
        outs[mode] = (tb.gmm(dev(a, cuda), dev(b, cuda)), tb.gmm(dev(an, cuda), dev(bn_, cuda)),
                      tb.gmm(dev(an, cuda), dev(bn_, cuda), out_f16=True, bias=bias, relu="gelu", residual=res),
                      tb.gmm(dev(an, cuda), dev(bn_, cuda), out_f16=True, bias=bias), acc)
    torch.cuda.synchronize()
    for mode in ("cta_group2",):
        for x, y in zip(outs["unpaired"], outs[mode]):
            assert torch.equal(x, y), mode
    rows = 128
    c = outs["cta_group2"][0].cpu().numpy()
    assert O.tensors_bitwise_equal(c[:rows], O.gmm(a[:rows], b, threads=8))
    assert O.tensors_bitwise_equal(c[-rows:], O.gmm(a[-rows:], b, threads=8))


def test_gmm_unsupported_and_value_errors(cuda):
    import torch

    a = torch.zeros(64, 12, device=cuda, dtype=torch.float16)
    b = torch.zeros(12, 64, device=cuda, dtype=torch.float16)
    with pytest.raises(tb.TirError) as e:
        tb.gmm(a, b)
    assert e.value.kind == "UnsupportedShape"
    with pytest.raises(tb.TirError) as e:
        tb.gmm(a.float(), b)
    assert e.value.kind == "ValueError"


def test_host_buffer_paths(cuda):
    M, N, K = 192, 64, 96
    a = O.reference_tensor((M, K), 1)
    b = O.reference_tensor((K, N), 2)
    want = O.gmm(a, b)
    assert O.tensors_bitwise_equal(tb.gmm_host(a.astype(np.float16), b.astype(np.float16)), want)
    assert O.tensors_bitwise_equal(tb.gmm_host(a, b), want)  # f32 storage of fp16 values
    c0 = O.reference_tensor((M, N), 3)
    got = tb.gmm_host(a, b, c0.copy(), accumulate=True)
    assert O.tensors_bitwise_equal(got, O.gmm(a, b, c0))
    spec = SMALL["GRP"]
    x = O.reference_tensor(spec.x_shape(), 4)
    w = O.reference_tensor(spec.w_shape(), 5)
    assert O.tensors_bitwise_equal(tb.conv_host(spec, x, w), O.conv(ospec(spec), x, w))


def test_inexact_fp16_input_rejected(cuda):
    a = np.full((128, 64), 0.1, np.float32)  # 0.1 is not an fp16 value
    b = np.ones((64, 64), np.float32)
    with pytest.raises(tb.TirError) as e:
        tb.gmm_host(a, b)
    assert e.value.kind == "ValueError" and "inexact" in e.value.message


def test_native_kernels_actually_launch(cuda):
    import torch

    tb.reset_launch_count()
    tb.gmm(torch.zeros(128, 64, device=cuda, dtype=torch.float16),
           torch.zeros(64, 64, device=cuda, dtype=torch.float16))
    spec = SMALL["DEP"]
    tb.conv(spec, torch.zeros(*spec.x_shape(), device=cuda, dtype=torch.float16),
            torch.zeros(*spec.w_shape(), device=cuda, dtype=torch.float16))
    torch.cuda.synchronize()
    assert tb.launch_count() == 2


@pytest.mark.parametrize("switch", [("no_halo", 1), ("no_tma_store", 1), ("epi8", 1), ("ks", 1), ("mc", 0),
                                    ("no_pdl", 1)], ids=lambda t: f"{t[0]}={t[1]}")
def test_planner_switches_exact(switch, option, cuda):
    """Planner switches (tir_b200_set_option) change tiling / epilogue flavour,
    never results: bit-exact on the reference distribution, with bias + ReLU and
    fp16 output, at the paper's C2D shape (sampled images) and a small wide shape."""
    import torch

    option(*switch)
    for spec in (tb.PAPER_SHAPES["C2D"], tb.Conv("C2D", n=2, in_dhw=(1, 5, 140), ci=64, co=64, k=(1, 3, 3),
                                                  p=(0, 1, 1))):
        x = O.reference_tensor(spec.x_shape(), 21)
        w = O.reference_tensor(spec.w_shape(), 22)
        bias = O.reference_tensor((spec.co,), 23)
        got = run_conv(spec, x, w, cuda)
        fused = tb.conv(spec, dev(x, cuda), dev(w, cuda), out_f16=True, bias=torch.from_numpy(bias).to(cuda),
                        relu=True).float().cpu().numpy()
        one = ospec(spec.with_(n=1))
        for img in (0, spec.n - 1):
            want = O.conv(one, x[img:img + 1], w, threads=8)
            assert O.tensors_bitwise_equal(got[img:img + 1], want), (switch, img)
            ref16 = np.maximum(want + bias, 0).astype(np.float16).astype(np.float32)
            assert np.array_equal(fused[img:img + 1], ref16), (switch, img)


def kernels_launched(fn):
    """Names of the CUDA kernels `fn` launches (torch profiler / CUPTI)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]


@pytest.mark.parametrize("name", ["C3D_rp", "C3D_rp_odd", "C2D_stem7", "C2D_stem3", "DIL_rp", "C2D_stem7_narrow",
                                  "C3D_rp_s1d"])
def test_rowpack_vs_im2col_exact(name, option, cuda):
    """The rowpack kernel (default for these shapes: A operand packed in TMEM) and the
    (kw, c) relayout + im2col path (no_rowpack = 1) both equal the oracle bit for bit."""
    spec = SMALL[name]
    x = O.reference_tensor(spec.x_shape(), 33)
    w = O.reference_tensor(spec.w_shape(), 34)
    want = O.conv(ospec(spec), x, w, threads=8)
    out = {}
    names = kernels_launched(lambda: out.setdefault("y", run_conv(spec, x, w, cuda)))
    assert any("conv_rowpack_kernel" in k for k in names), names
    assert O.tensors_bitwise_equal(out["y"], want)
    option("no_rowpack", 1)
    out = {}
    names = kernels_launched(lambda: out.setdefault("y", run_conv(spec, x, w, cuda)))
    assert not any("conv_rowpack_kernel" in k for k in names), names
    assert O.tensors_bitwise_equal(out["y"], want)


@pytest.mark.parametrize("name", ["GRP", "GRP_gp16", "GRP_gp32"])
def test_group_packed_vs_per_group_exact(name, option, cuda):
    """The group-packed igemm (default for 16 / 32 channels per group, 32 per output
    group) and the per-group narrow-piece plan (no_gpack = 1) both equal the oracle
    bit for bit; the packed plan launches the GP instantiation."""
    spec = SMALL[name]
    x = O.reference_tensor(spec.x_shape(), 35)
    w = O.reference_tensor(spec.w_shape(), 36)
    want = O.conv(ospec(spec), x, w, threads=8)
    out = {}
    names = kernels_launched(lambda: out.setdefault("y", run_conv(spec, x, w, cuda)))
    assert any("igemm_tc_kernel" in k and k.rstrip(">)").count("true") for k in names), names
    assert O.tensors_bitwise_equal(out["y"], want)
    option("no_gpack", 1)
    out = {}
    run = run_conv(spec, x, w, cuda)
    assert O.tensors_bitwise_equal(run, want)


@pytest.mark.parametrize("name", ["DIL", "C3D"])
def test_opt_in_pack_hw_exact(name, option, cuda):
    """The opt-in (kh, kw, c) relayout (pack_hw = 1) stays bit-exact."""
    option("pack_hw", 1)
    spec = SMALL[name]
    x = O.reference_tensor(spec.x_shape(), 31)
    w = O.reference_tensor(spec.w_shape(), 32)
    got = run_conv(spec, x, w, cuda)
    assert O.tensors_bitwise_equal(got, O.conv(ospec(spec), x, w, threads=8))


def test_host_path_batch_pipeline_exact(cuda):
    """tir_b200_conv_host splits the batch into chunks pipelined over three
    streams (H2D / conv / D2H overlap): uneven chunks, accumulate, bit-exact."""
    spec = tb.Conv("C2D", n=5, in_dhw=(1, 9, 11), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1))
    x = O.reference_tensor(spec.x_shape(), 41)
    w = O.reference_tensor(spec.w_shape(), 42)
    y0 = O.reference_tensor(spec.y_shape(), 43)
    want = O.conv(ospec(spec), x, w, threads=8)
    got = tb.conv_host(spec, x.astype(np.float16), w.astype(np.float16))
    assert O.tensors_bitwise_equal(got, want)
    acc = tb.conv_host(spec, x.astype(np.float16), w.astype(np.float16), y0.copy(), accumulate=True)
    assert O.tensors_bitwise_equal(acc, O.conv(ospec(spec), x, w, y0, threads=8))
