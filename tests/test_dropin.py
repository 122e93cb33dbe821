"""Drop-in tests: the reference interpreter (tir::run, unchanged, built from
/root/reference into oracle/_ref) dispatches tensorized blocks to the B200
kernels through HostKernels registered by paper_2207_04296_b200/adapter/.

Mirrors the reference's own intrinsic tests (tests/test_interp.cc:162-227):
tiled accumulate semantics with intrinsic_calls == 8, DuplicateName on
re-registration, UnregisteredIntrinsic for unknown names — with the B200
kernel as the "virtual accelerator".
"""
import ctypes
import os

import numpy as np
import pytest

from oracle import ir_gen as G
from oracle import oracle as O
from paper_2207_04296_b200 import api

pytestmark = pytest.mark.gpu

ADAPTER = os.path.join(os.path.dirname(api.LIB_PATH), "libtir_b200_adapter.so")


def adapter():
    if not os.path.exists(ADAPTER):
        pytest.fail("adapter library not built (needs /root/reference at build time)")
    L = ctypes.CDLL(ADAPTER)
    f32p = ctypes.POINTER(ctypes.c_float)
    L.tir_b200_adapter_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(api.ConvDesc),
                                       ctypes.c_int, ctypes.POINTER(f32p), f32p, ctypes.c_int64,
                                       ctypes.POINTER(ctypes.c_int64), ctypes.c_char_p, ctypes.c_int]
    return L


def run(ir, intrin, inputs, out_shape, desc=None):
    L = adapter()
    ins = [np.ascontiguousarray(x, np.float32) for x in inputs]
    arr = (ctypes.POINTER(ctypes.c_float) * len(ins))(*[x.ctypes.data_as(ctypes.POINTER(ctypes.c_float)) for x in ins])
    out = np.zeros(out_shape, np.float32)
    calls = ctypes.c_int64(0)
    err = ctypes.create_string_buffer(1024)
    rc = L.tir_b200_adapter_run(ir.encode(), intrin.encode(), ctypes.byref(desc) if desc else None,
                                len(ins), arr, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                out.size, ctypes.byref(calls), err, 1024)
    if rc != 0:
        kind, _, msg = err.value.decode().partition("|")
        raise api.TirError(kind, msg)
    return out, calls.value


def test_whole_op_gmm_block(cuda):
    M, N, K = 256, 128, 192
    a = O.reference_tensor((M, K), 1)
    b = O.reference_tensor((K, N), 2)
    out, calls = run(G.tensorized_gmm_source(M, N, K), "b200.gmm", [a, b], (M, N))
    assert calls == 1
    assert O.tensors_bitwise_equal(out, O.gmm(a, b))


def test_tiled_gmm_blocks_accumulate(cuda):
    # 2x2x2 tiles like the reference's accel.dot test: 8 intrinsic calls, each
    # accumulating into its C window (blockize semantics, schedule_block.cc:570-603)
    M, N, K = 256, 128, 256
    a = O.reference_tensor((M, K), 3)
    b = O.reference_tensor((K, N), 4)
    out, calls = run(G.tensorized_gmm_source(M, N, K, tiles=(2, 2, 2)), "b200.gmm", [a, b], (M, N))
    assert calls == 8
    assert O.tensors_bitwise_equal(out, O.gmm(a, b))


def test_dropin_matches_scalar_program(cuda):
    # same inputs, the scalar reference program vs the tensorized B200 program
    M, N, K = 128, 64, 64
    a = O.normal_f16((M, K), 5)
    b = O.normal_f16((K, N), 6)
    scalar, _ = O.ref_run(G.gmm_source(M, N, K), [a, b], (M, N))
    tensorized, _ = run(G.tensorized_gmm_source(M, N, K), "b200.gmm", [a, b], (M, N))
    assert O.tensors_close_dot(tensorized, scalar, O.gmm(np.abs(a), np.abs(b)), 1e-4, 1e-6)


@pytest.mark.parametrize("op", ["C2D", "GRP", "T2D", "DEP", "C1D", "DIL"])
def test_whole_op_conv_block(op, cuda):
    small = {
        "C2D": G.ConvSpec("C2D", n=2, in_dhw=(1, 9, 9), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1)),
        "GRP": G.ConvSpec("GRP", n=1, in_dhw=(1, 8, 8), ci=64, co=128, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=4),
        "T2D": G.ConvSpec("T2D", n=1, in_dhw=(1, 4, 4), ci=64, co=64, k=(1, 4, 4), s=(1, 2, 2), p=(0, 1, 1), transposed=True),
        "DEP": G.ConvSpec("DEP", n=1, in_dhw=(1, 10, 10), ci=32, co=32, k=(1, 3, 3), p=(0, 1, 1), groups=32),
        "C1D": G.ConvSpec("C1D", n=2, in_dhw=(1, 1, 20), ci=64, co=128, k=(1, 1, 3), s=(1, 1, 2), p=(0, 0, 1)),
        "DIL": G.ConvSpec("DIL", n=1, in_dhw=(1, 16, 16), ci=3, co=64, k=(1, 7, 7), s=(1, 2, 2), p=(0, 3, 3), d=(1, 2, 2)),
    }
    spec = small[op]
    x = O.reference_tensor(spec.x_shape(), 7)
    w = O.reference_tensor(spec.w_shape(), 8)
    desc = O.ConvDesc.from_spec(spec)
    d = api.ConvDesc(*[getattr(desc, f) for f, _ in O.ConvDesc._fields_])
    intrin = f"b200.{op.lower()}"
    out, calls = run(G.tensorized_conv_source(spec, intrin), intrin, [x, w], spec.y_shape(), desc=d)
    assert calls == 1
    assert O.tensors_bitwise_equal(out, O.conv(spec, x, w))


def test_unregistered_intrinsic_kind(cuda):
    M = N = K = 64
    with pytest.raises(api.TirError) as e:
        run(G.tensorized_gmm_source(M, N, K, intrin="b200.nosuch"), "b200.gmm",
            [np.zeros((M, K)), np.zeros((K, N))], (M, N))
    assert e.value.kind == "UnregisteredIntrinsic"


def test_view_mismatch_is_value_error(cuda):
    spec = G.ConvSpec("C2D", n=1, in_dhw=(1, 8, 8), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1))
    other = G.ConvSpec("C2D", n=1, in_dhw=(1, 8, 8), ci=64, co=64, k=(1, 3, 3), p=(0, 0, 0))
    desc = O.ConvDesc.from_spec(other)
    d = api.ConvDesc(*[getattr(desc, f) for f, _ in O.ConvDesc._fields_])
    with pytest.raises(api.TirError) as e:
        run(G.tensorized_conv_source(spec, "b200.c2d"), "b200.c2d",
            [np.zeros(spec.x_shape()), np.zeros(spec.w_shape())], spec.y_shape(), desc=d)
    assert e.value.kind == "ValueError"


def test_inexact_input_through_interpreter(cuda):
    M = N = K = 64
    a = np.full((M, K), 1.0 / 3.0, np.float32)
    with pytest.raises(api.TirError) as e:
        run(G.tensorized_gmm_source(M, N, K), "b200.gmm", [a, np.ones((K, N))], (M, N))
    assert e.value.kind == "ValueError"


def run_scalar(ir, intrin, desc, params, inputs, out_shape):
    L = adapter()
    f32p = ctypes.POINTER(ctypes.c_float)
    L.tir_b200_adapter_run_scalar.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                              ctypes.c_int, ctypes.POINTER(f32p), f32p, ctypes.c_int64,
                                              ctypes.POINTER(ctypes.c_int64), ctypes.c_char_p, ctypes.c_int]
    ins = [np.ascontiguousarray(x, np.float32) for x in inputs]
    arr = (f32p * len(ins))(*[x.ctypes.data_as(f32p) for x in ins])
    out = np.zeros(out_shape, np.float32)
    calls = ctypes.c_int64(0)
    err = ctypes.create_string_buffer(1024)
    rc = L.tir_b200_adapter_run_scalar(ir.encode(), intrin.encode(), desc.encode(), params.encode(), len(ins), arr,
                                       out.ctypes.data_as(f32p), out.size, ctypes.byref(calls), err, 1024)
    if rc != 0:
        kind, _, msg = err.value.decode().partition("|")
        raise api.TirError(kind, msg)
    return out, calls.value


def _desc(src: str) -> str:
    """A description PrimFunc: the scalar program without its init (an intrinsic
    ACCUMULATES into its output window, interp.cc:594-726 runs only the body)."""
    import re

    return re.sub(r"init \{[^}]*\}\s*", "", src)


@pytest.mark.parametrize("dist", ["D1", "D2"])
def test_per_call_parity_vs_reference_scalar_kernel_gmm(dist, cuda):
    """every intrinsic CALL of a tiled program (8 calls of a
    64x64x64 GEMM tile, accumulating over the K tiles) computed by the B200
    HostKernel equals the reference's own scalar implementation of that
    intrinsic, make_scalar_kernel(desc) (interp.cc:594-726), registered under
    the same name: bit-exact on D1, within the D2 bar on N(0,1) fp16."""
    M = N = K = 128
    gen = O.reference_tensor if dist == "D1" else O.normal_f16
    a, b = gen((M, K), 1), gen((K, N), 2)
    ir = G.tensorized_gmm_source(M, N, K, tiles=(2, 2, 2))
    gpu, calls = run(ir, "b200.gmm", [a, b], (M, N))
    ref, calls_ref = run_scalar(ir, "b200.gmm", _desc(G.gmm_source(64, 64, 64)), "C,A,B", [a, b], (M, N))
    assert calls == calls_ref == 8
    if dist == "D1":
        assert O.tensors_bitwise_equal(gpu, ref)
    else:
        abs_sum = O.gmm(np.abs(a), np.abs(b))
        assert O.tensors_close_dot(gpu, ref, abs_sum, 1e-4, 1e-6)


@pytest.mark.parametrize("op", ["C2D", "GRP", "C1D"])
def test_per_call_parity_vs_reference_scalar_kernel_conv(op, cuda):
    """The whole-op conv intrinsic against make_scalar_kernel of its own
    description (the unpadded conv block: the scalar kernel evaluates loads,
    casts and arithmetic only, no select), bit-exact on D1."""
    specs = {"C2D": G.ConvSpec("C2D", n=2, in_dhw=(1, 10, 9), ci=64, co=32, k=(1, 3, 3)),
             "GRP": G.ConvSpec("GRP", n=1, in_dhw=(1, 8, 8), ci=64, co=64, k=(1, 3, 3), groups=2),
             "C1D": G.ConvSpec("C1D", n=2, in_dhw=(1, 1, 20), ci=64, co=64, k=(1, 1, 3), s=(1, 1, 2))}
    spec = specs[op]
    x = O.reference_tensor(spec.x_shape(), 3)
    w = O.reference_tensor(spec.w_shape(), 4)
    d = api.ConvDesc(api.OP_CODES[op], 0, spec.n, *spec.in_dhw, spec.ci, spec.co, *spec.k, *spec.s, *spec.p,
                     *spec.d, spec.groups)
    intrin = f"b200.{op.lower()}"
    ir = G.tensorized_conv_source(spec, intrin)
    gpu, _ = run(ir, intrin, [x, w], spec.y_shape(), desc=d)
    ref, _ = run_scalar(ir, intrin, _desc(G.conv_source(spec)), "C,A,B", [x, w], spec.y_shape())
    assert O.tensors_bitwise_equal(gpu, ref)
    assert O.tensors_bitwise_equal(ref, O.conv(spec, x, w))
