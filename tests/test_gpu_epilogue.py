"""GPU parity for the golden vectors and the fused epilogue.

* Every case in tests/golden (made by the reference interpreter, tir::run) runs
  through the C-ABI on the GPU: D1 cases bit-exact, D2 cases within the
  test_gpu_parity tolerances. That includes the reference's own matmul16 /
  conv2d / depthwise / gemm_relu programs (tests/testing/workloads.h).
* Epilogue variants (bias, relu, both; with accumulate; with fp16 output) on
  every kernel path: halo TMA store, halo direct store (in-place accumulate),
  im2col TMA store, im2col generic store (T2D scatter, accumulate), (kw, c)
  packing, grouped channel padding, DEP tile kernel, DEP generic kernel, GMM
  (where split-K is disabled by the epilogue). D1 bit-exact against
  oracle.epilogue(oracle.conv/gmm(...)).
"""
import numpy as np
import pytest

import paper_2207_04296_b200 as tb
from oracle import oracle as O

from test_gpu_parity import DOT_TOL_D2, REL_TOL_D2, SMALL, dev, ospec

pytestmark = pytest.mark.gpu


def _conv_spec(meta) -> tb.Conv:
    s = dict(meta["spec"])
    return tb.Conv(s["op"], n=s["n"], in_dhw=tuple(s["in_dhw"]), ci=s["ci"], co=s["co"], k=tuple(s["k"]),
                   s=tuple(s["s"]), p=tuple(s["p"]), d=tuple(s["d"]), groups=s["groups"],
                   transposed=s["transposed"])


_OWN = {
    "conv2d": tb.Conv("C2D", n=1, in_dhw=(1, 8, 8), ci=4, co=8, k=(1, 3, 3)),
    "depthwise": tb.Conv("DEP", n=1, in_dhw=(1, 8, 8), ci=8, co=8, k=(1, 3, 3), groups=8),
}


def _golden_names():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")) as f:
        return list(json.load(f))


def _bias(arrays, name, cuda):
    import torch

    b = arrays.get(f"{name}/bias")
    return None if b is None else torch.from_numpy(np.ascontiguousarray(b, np.float32)).to(cuda)


@pytest.mark.parametrize("name", _golden_names())
def test_golden_vector_on_gpu(golden, name, cuda):
    import torch

    meta, arrays = golden
    m = meta[name]
    a, b, want = arrays[f"{name}/a"], arrays[f"{name}/b"], arrays[f"{name}/out"]
    epi = m.get("epilogue", {"bias": False, "relu": False})
    kw = {"bias": _bias(arrays, name, cuda) if epi["bias"] else None, "relu": epi["relu"]}
    kind = m["kind"] if m["kind"] != "reference_workload" else m["source"][0]
    if kind in ("gmm", "matmul", "gemm_relu"):
        got = tb.gmm(dev(a, cuda), dev(b, cuda), **kw)
    else:
        spec = _conv_spec(m) if kind == "conv" else _OWN[kind]
        got = tb.conv(spec, dev(a, cuda), dev(b, cuda), **kw)
    torch.cuda.synchronize()
    got = got.float().cpu().numpy()
    assert got.shape == want.shape
    if m.get("dist", "D1") == "D1":
        assert O.tensors_bitwise_equal(got, want), f"max diff {np.abs(got - want).max()}"
    else:
        spec = _conv_spec(m)
        absum = O.conv(ospec(spec), np.abs(a), np.abs(b))
        assert O.tensors_close_dot(got, want, absum, REL_TOL_D2, DOT_TOL_D2)


EPI_CASES = ["C1D", "C2D", "C2D_ci96_co40", "C2D_ci8", "C3D", "DIL", "GRP", "GRP_g2", "T2D", "DEP",
             "DEP_s2", "DEP_c12", "C3D_rp", "C2D_stem7", "C2D_stem3", "DIL_rp"]
VARIANTS = [(True, False), (False, True), (True, True)]


def _epi_inputs(spec, seed=1):
    x = O.reference_tensor(spec.x_shape(), seed)
    w = O.reference_tensor(spec.w_shape(), seed + 1)
    bias = O.reference_tensor((spec.co,), seed + 2)
    return x, w, bias


@pytest.mark.parametrize("bias_on,relu", VARIANTS)
@pytest.mark.parametrize("name", EPI_CASES)
def test_conv_epilogue_bit_exact(name, bias_on, relu, cuda):
    import torch

    spec = SMALL[name]
    x, w, bias = _epi_inputs(spec)
    bt = torch.from_numpy(bias).to(cuda) if bias_on else None
    got = tb.conv(spec, dev(x, cuda), dev(w, cuda), bias=bt, relu=relu)
    torch.cuda.synchronize()
    want = O.epilogue(O.conv(ospec(spec), x, w, threads=8), bias if bias_on else None, relu)
    assert O.tensors_bitwise_equal(got.cpu().numpy(), want), name


@pytest.mark.parametrize("name", ["C2D", "C2D_ci96_co40", "GRP", "T2D", "DEP", "DEP_c12", "C2D_stem7", "C2D_stem3"])
def test_conv_epilogue_with_accumulate_and_fp16(name, cuda):
    import torch

    spec = SMALL[name]
    x, w, bias = _epi_inputs(spec, 5)
    yin = O.reference_tensor(spec.y_shape(), 9)
    bt = torch.from_numpy(bias).to(cuda)
    want = O.epilogue(O.conv(ospec(spec), x, w, yin, threads=8), bias, True)
    # in place (Y is Yin): the halo / im2col paths cannot use TMA reduce-add here
    y = torch.from_numpy(yin.copy()).to(cuda)
    tb.conv(spec, dev(x, cuda), dev(w, cuda), y, accumulate=True, bias=bt, relu=True)
    torch.cuda.synchronize()
    assert O.tensors_bitwise_equal(y.cpu().numpy(), want), name
    # fp16 output = RN(fp32 epilogue result)
    y16 = tb.conv(spec, dev(x, cuda), dev(w, cuda), out_f16=True, bias=bt, relu=True)
    torch.cuda.synchronize()
    want16 = O.epilogue(O.conv(ospec(spec), x, w, threads=8), bias, True).astype(np.float16)
    assert np.array_equal(y16.cpu().numpy().view(np.uint16), want16.view(np.uint16)), name


@pytest.mark.parametrize("mnk", [(16, 16, 16), (128, 64, 64), (200, 72, 128), (256, 256, 512),
                                 (1024, 1024, 1024)])
@pytest.mark.parametrize("bias_on,relu", VARIANTS)
def test_gmm_epilogue_bit_exact(mnk, bias_on, relu, cuda):
    import torch

    m, n, k = mnk
    a = O.reference_tensor((m, k), 3)
    b = O.reference_tensor((k, n), 4)
    bias = O.reference_tensor((n,), 5)
    bt = torch.from_numpy(bias).to(cuda) if bias_on else None
    got = tb.gmm(dev(a, cuda), dev(b, cuda), bias=bt, relu=relu)
    torch.cuda.synchronize()
    want = O.epilogue(O.gmm(a, b, threads=8), bias if bias_on else None, relu)
    assert O.tensors_bitwise_equal(got.cpu().numpy(), want)
    # accumulate into a separate-but-aliased C (generic store path)
    c0 = O.reference_tensor((m, n), 6)
    c = torch.from_numpy(c0.copy()).to(cuda)
    tb.gmm(dev(a, cuda), dev(b, cuda), c, accumulate=True, bias=bt, relu=relu)
    torch.cuda.synchronize()
    want = O.epilogue(O.gmm(a, b, c0, threads=8), bias if bias_on else None, relu)
    assert O.tensors_bitwise_equal(c.cpu().numpy(), want)


@pytest.mark.parametrize("name,act", [("C2D_stem7", "relu"), ("C2D_stem3", "relu6"), ("C3D_rp", "gelu")])
def test_rowpack_fused_stem_epilogue(name, act, cuda):
    """The network stems' fused form on the rowpack kernel: bias + activation with
    fp16 output, bit-exact against oracle.epilogue of the fp32 result, RN to fp16."""
    import torch

    spec = SMALL[name]
    x, w, bias = _epi_inputs(spec, seed=7)
    got = tb.conv(spec, dev(x, cuda), dev(w, cuda), bias=torch.from_numpy(bias).to(cuda), relu=act, out_f16=True)
    torch.cuda.synchronize()
    pre = O.epilogue(O.conv(ospec(spec), x, w, threads=8), bias)  # f32: conv + bias
    got = got.float().cpu().numpy()
    if act == "relu":
        want = np.where(pre < 0, np.float32(0), pre)
    elif act == "relu6":
        want = np.minimum(np.where(pre < 0, np.float32(0), pre), np.float32(6))
    else:  # erf GELU, float64 reference; the kernel's erf approximation is within 1.5e-7
        from math import erf
        want = np.vectorize(lambda v: 0.5 * v * (1.0 + erf(v / 2 ** 0.5)))(pre.astype(np.float64))
    want = want.astype(np.float16).astype(np.float32)
    if act == "gelu":
        assert np.allclose(got, want, rtol=2 ** -10, atol=1e-3)
    else:
        assert np.array_equal(got, want)


def test_epilogue_d2_relu_matches_sign_of_result(cuda):
    """D2 (fp16 normals): with relu, every output is max(conv, 0) of the
    no-epilogue kernel result bit for bit (the epilogue is applied to the same
    accumulator), and bias adds exactly once."""
    import torch

    spec = SMALL["C2D"]
    x = O.normal_f16(spec.x_shape(), 1)
    w = O.normal_f16(spec.w_shape(), 2)
    bias = O.normal_f16((spec.co,), 3)
    X, W = dev(x, cuda), dev(w, cuda)
    plain = tb.conv(spec, X, W).cpu().numpy()
    fused = tb.conv(spec, X, W, bias=torch.from_numpy(bias).to(cuda), relu=True).cpu().numpy()
    assert O.tensors_bitwise_equal(fused, O.epilogue(plain, bias, True))


def test_epilogue_argument_errors(cuda):
    import torch

    spec = SMALL["C2D"]
    x, w, _ = _epi_inputs(spec)
    with pytest.raises(tb.TirError) as e:
        tb.conv(spec, dev(x, cuda), dev(w, cuda), bias=torch.zeros(spec.co + 1, device=cuda))
    assert e.value.kind == "ValueError"
    with pytest.raises(tb.TirError):
        tb.conv(spec, dev(x, cuda), dev(w, cuda), bias=torch.zeros(spec.co, device=cuda).half())
