"""CPU tests: the oracle is pinned before it is trusted.

  * the C restatement (oracle/tir_oracle.c) reproduces every golden vector the
    reference interpreter produced (tests/golden, made by make_golden.py),
    including the reference's own workload programs (test_interp.cc:29-73);
  * our Python port of random_tensor (workloads.h:170-184) equals the
    reference's generator;
  * where the reference is built (this container), a sweep of fresh shapes
    runs through tir::run and the restatement and must agree bit-for-bit;
  * an independent float64 torch computation agrees exactly on the reference
    distribution (every partial sum is exact).
"""
import os

import numpy as np
import pytest

from oracle import ir_gen as G
from oracle import oracle as O


def _spec(meta):
    s = dict(meta["spec"])
    for k in ("in_dhw", "k", "s", "p", "d"):
        s[k] = tuple(s[k])
    return G.ConvSpec(**s)


def test_golden_cases_present(golden):
    meta, arrays = golden
    ops = {m["spec"]["op"] for m in meta.values() if m["kind"] == "conv"}
    assert ops == {"C1D", "C2D", "C3D", "DIL", "GRP", "T2D", "DEP"}
    assert any(m["kind"] == "gmm" for m in meta.values())
    assert {"ref_matmul16", "ref_conv2d", "ref_depthwise"} <= set(meta)


def test_restatement_matches_reference_golden(golden):
    meta, arrays = golden
    for name, m in meta.items():
        a, b, want = arrays[f"{name}/a"], arrays[f"{name}/b"], arrays[f"{name}/out"]
        if m["kind"] == "gmm":
            got = O.gmm(a, b)
        elif m["kind"] == "conv":
            got = O.conv(_spec(m), a, b)
        else:  # the reference's own workload programs
            which = m["source"][0]
            if which in ("matmul", "gemm_relu"):
                got = O.gmm(a, b)
            elif which == "conv2d":
                spec = G.ConvSpec("C2D", n=1, in_dhw=(1, 8, 8), ci=4, co=8, k=(1, 3, 3))
                got = O.conv(spec, a, b)
            else:
                spec = G.ConvSpec("DEP", n=1, in_dhw=(1, 8, 8), ci=8, co=8, k=(1, 3, 3), groups=8)
                got = O.conv(spec, a, b)
        if "epilogue" in m:
            got = O.epilogue(got, arrays.get(f"{name}/bias") if m["epilogue"]["bias"] else None,
                             m["epilogue"]["relu"])
        assert got.shape == want.shape, name
        assert O.tensors_bitwise_equal(got, want), name


def test_golden_epilogue_cases_present(golden):
    meta, _ = golden
    epi = {k for k, m in meta.items() if "epilogue" in m}
    assert "ref_gemm_relu16" in epi  # the reference's own gemm_relu_source program
    assert len(epi) >= 5


@pytest.mark.skipif(not O.ref_available(), reason="reference interpreter not built")
@pytest.mark.parametrize("bias,relu", [(True, False), (False, True), (True, True)])
def test_epilogue_oracle_matches_reference_interpreter(bias, relu):
    """ir_gen.with_epilogue programs through tir::run vs oracle conv + epilogue,
    on D2 (fp16 normals) where bias + relu see both signs and exact zeros."""
    spec = G.ConvSpec("C2D", n=1, in_dhw=(1, 5, 6), ci=8, co=16, k=(1, 3, 3), p=(0, 1, 1))
    x, w = O.normal_f16(spec.x_shape(), 31), O.normal_f16(spec.w_shape(), 32)
    bvec = O.normal_f16((spec.co,), 33)
    ins = [x, w] + ([bvec] if bias else [])
    src = G.with_epilogue(G.conv_source(spec), spec.y_shape(), bias, relu)
    want, _ = O.ref_run(src, ins, spec.y_shape())
    got = O.epilogue(O.conv(spec, x, w), bvec if bias else None, relu)
    assert O.tensors_bitwise_equal(got, want)


def test_random_tensor_port_matches_reference_inputs(golden):
    meta, arrays = golden
    # ref_matmul16 inputs were drawn by the reference's random_tensor with seeds 1, 2
    np.testing.assert_array_equal(O.reference_tensor((16, 16), 1), arrays["ref_matmul16/a"])
    np.testing.assert_array_equal(O.reference_tensor((16, 16), 2), arrays["ref_matmul16/b"])
    np.testing.assert_array_equal(O.reference_tensor((1, 8, 8, 8), 9), arrays["ref_depthwise/a"])


def test_reference_distribution_is_fp16_exact():
    x = O.reference_tensor((4096,), 5)
    assert np.array_equal(x.astype(np.float16).astype(np.float32), x)
    assert set(np.unique(x * 8 + 32).astype(int)) <= set(range(64))


def test_multithreaded_oracle_is_deterministic():
    spec = G.ConvSpec("C2D", n=3, in_dhw=(1, 9, 7), ci=8, co=8, k=(1, 3, 3), p=(0, 1, 1))
    x = O.normal_f16(spec.x_shape(), 1)
    w = O.normal_f16(spec.w_shape(), 2)
    a = O.conv(spec, x, w, threads=1)
    b = O.conv(spec, x, w, threads=7)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_accumulate_semantics():
    a = O.reference_tensor((8, 8), 20)
    b = O.reference_tensor((8, 8), 21)
    c0 = O.reference_tensor((8, 8), 22)
    assert O.tensors_bitwise_equal(O.gmm(a, b, c0), c0 + O.gmm(a, b))


def _torch_conv64(spec, x, w):
    import torch
    import torch.nn.functional as F

    r = spec.spatial_rank
    X = torch.from_numpy(x.astype(np.float64))
    if spec.op == "DEP":
        W = torch.from_numpy(w.astype(np.float64)).unsqueeze(-2)  # [K.., 1, C]
    else:
        W = torch.from_numpy(w.astype(np.float64))
    # channels-last -> channels-first
    perm_x = (0, r + 1, *range(1, r + 1))
    X = X.permute(*perm_x)
    k_sp = spec.k[3 - r:]
    s, p, d = spec.s[3 - r:], spec.p[3 - r:], spec.d[3 - r:]
    if spec.transposed:
        # ours: W[k.., ci, co]; torch conv_transpose: [ci, co, k..]
        Wt = W.permute(r, r + 1, *range(r))
        fn = {1: F.conv_transpose1d, 2: F.conv_transpose2d, 3: F.conv_transpose3d}[r]
        Y = fn(X, Wt, stride=s, padding=p, dilation=d, groups=spec.groups)
    else:
        Wt = W.permute(r + 1, r, *range(r))  # [co, ci/g, k..]
        fn = {1: F.conv1d, 2: F.conv2d, 3: F.conv3d}[r]
        Y = fn(X, Wt, stride=s, padding=p, dilation=d, groups=spec.groups)
    del k_sp
    return Y.permute(0, *range(2, r + 2), 1).numpy()


@pytest.mark.parametrize("name", ["C1D", "C2D", "C2D_s2", "C3D", "DIL", "GRP", "T2D", "DEP", "DEP_s2"])
def test_independent_torch_float64_agrees_exactly(golden, name):
    meta, arrays = golden
    spec = _spec(meta[name])
    want = arrays[f"{name}/out"].astype(np.float64)
    got = _torch_conv64(spec, arrays[f"{name}/a"], arrays[f"{name}/b"])
    assert got.shape == want.shape
    np.testing.assert_array_equal(got, want)


SWEEP = [
    G.ConvSpec("C2D", n=2, in_dhw=(1, 5, 7), ci=8, co=8, k=(1, 3, 2), s=(1, 2, 1), p=(0, 1, 0)),
    G.ConvSpec("C2D", n=1, in_dhw=(1, 6, 6), ci=4, co=4, k=(1, 1, 1)),
    G.ConvSpec("DIL", n=1, in_dhw=(1, 10, 8), ci=4, co=4, k=(1, 3, 3), d=(1, 3, 2), p=(0, 3, 2)),
    G.ConvSpec("GRP", n=2, in_dhw=(1, 5, 5), ci=8, co=4, k=(1, 3, 3), p=(0, 1, 1), groups=2),
    G.ConvSpec("T2D", n=1, in_dhw=(1, 3, 4), ci=4, co=4, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), transposed=True),
    G.ConvSpec("T2D", n=1, in_dhw=(1, 2, 2), ci=4, co=4, k=(1, 4, 4), s=(1, 2, 2), p=(0, 0, 0), transposed=True),
    G.ConvSpec("C1D", n=3, in_dhw=(1, 1, 9), ci=4, co=4, k=(1, 1, 5), s=(1, 1, 3), p=(0, 0, 2)),
    G.ConvSpec("C3D", n=1, in_dhw=(3, 4, 4), ci=2, co=4, k=(2, 3, 3), s=(1, 1, 2), p=(0, 1, 1)),
    G.ConvSpec("DEP", n=1, in_dhw=(1, 7, 5), ci=4, co=4, k=(1, 5, 3), s=(1, 2, 1), p=(0, 2, 1), groups=4),
]


@pytest.mark.skipif(not O.ref_available(), reason="reference interpreter not built (oracle/_ref)")
@pytest.mark.parametrize("spec", SWEEP, ids=lambda s: s.op)
def test_restatement_matches_tir_run_sweep(spec):
    x = O.normal_f16(spec.x_shape(), 31)
    w = O.normal_f16(spec.w_shape(), 32)
    want, _ = O.ref_run(G.conv_source(spec), [x, w], spec.y_shape())
    got = O.conv(spec, x, w)
    assert np.array_equal(want.view(np.uint32), got.view(np.uint32))


@pytest.mark.skipif(not O.ref_available(), reason="reference interpreter not built (oracle/_ref)")
def test_row_and_column_slices_are_bit_identical():
    spec = G.ConvSpec("C2D", n=2, in_dhw=(1, 6, 6), ci=4, co=4, k=(1, 3, 3), p=(0, 1, 1))
    x = O.normal_f16(spec.x_shape(), 1)
    w = O.normal_f16(spec.w_shape(), 2)
    full = O.conv(spec, x, w)
    part, _ = O.ref_run(G.conv_source(spec, rows=(7, 9), cols=(2, 5)), [x, w], spec.y_shape())
    n_h = spec.out_dhw()[1]
    for row in (7, 8):
        n, h = divmod(row, n_h)
        assert np.array_equal(part[n, h, 2:5], full[n, h, 2:5])


@pytest.mark.skipif(not O.ref_available(), reason="reference interpreter not built (oracle/_ref)")
def test_gmm_source_matches_tir_run():
    a = O.normal_f16((12, 20), 1)
    b = O.normal_f16((20, 16), 2)
    want, _ = O.ref_run(G.gmm_source(12, 16, 20), [a, b], (12, 16))
    assert np.array_equal(want.view(np.uint32), O.gmm(a, b).view(np.uint32))


def test_paper_shapes_flops():
    # SURVEY §8(d) table (GFLOP, algorithmic)
    want = {"C1D": 0.101, "C2D": 3.699, "C3D": 211.5, "DIL": 3.577, "GRP": 0.462, "T2D": 1.074,
            "DEP": 0.116}
    for op, g in want.items():
        assert abs(G.PAPER_SHAPES[op].flops() / 1e9 - g) / g < 0.01, op


def test_oracle_rejects_bad_geometry():
    with pytest.raises(ValueError):
        O.conv(G.ConvSpec("C2D", n=1, in_dhw=(1, 2, 2), ci=4, co=4, k=(1, 5, 5)),
               np.zeros((1, 2, 2, 4), np.float32), np.zeros((5, 5, 4, 4), np.float32))


def test_oracle_lib_has_no_gpu_dependency():
    import subprocess

    out = subprocess.run(["ldd", O.ORACLE_LIB], capture_output=True, text=True).stdout
    assert "cuda" not in out.lower()
    assert os.path.exists(O.ORACLE_LIB)
