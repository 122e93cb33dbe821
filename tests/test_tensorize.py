"""Caller-side whole-op tensorize composite.

paper_2207_04296_b200/adapter/tir_b200_tensorize.cc turns an unchanged scalar
workload PrimFunc into a program whose contraction block calls a B200
intrinsic, using only the reference's schedule API: Schedule::blockize
(src/schedule_block.cc:407-610), then Schedule::commit_rewrite with the step
"b200.tensorize" (schedule.cc:348-352), replayable through
register_step_handler (schedule.cc:354-363, apply_step :760-766).

CPU tests (the transform needs no GPU): the matcher recovers the exact
geometry of every op of the paper's set from the scalar program (the
characteristic-vector test of SPEC.md "propose_mapping" plus the affine input
index), the result is validate_all-clean and trace replay reproduces it, and
non-contractions / partial nests are rejected with the reference's error
style. GPU tests: tir::run of the tensorized program matches the oracle bit for
bit with one intrinsic call, including the reference's own gemm_relu program
(tensorized gemm + scalar relu block).
"""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import ir_gen as G
from oracle import oracle as O
from paper_2207_04296_b200 import api

ADAPTER = os.path.join(os.path.dirname(api.LIB_PATH), "libtir_b200_adapter.so")
OPS = {"GMM": 0, "C1D": 1, "C2D": 2, "C3D": 3, "DIL": 4, "GRP": 5, "T2D": 6, "DEP": 7}


def adapter():
    if not os.path.exists(ADAPTER):
        pytest.skip("adapter library not built (needs /root/reference at build time)")
    L = ctypes.CDLL(ADAPTER)
    f32p = ctypes.POINTER(ctypes.c_float)
    L.tir_b200_adapter_tensorize.argtypes = [
        ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64,
        ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(api.ConvDesc), ctypes.POINTER(ctypes.c_int64),
        ctypes.c_char_p, ctypes.c_int]
    L.tir_b200_adapter_run_auto.argtypes = [
        ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int, ctypes.c_int, ctypes.POINTER(f32p),
        f32p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), ctypes.c_char_p, ctypes.c_int]
    return L


def _raise(err):
    kind, _, msg = err.value.decode().partition("|")
    raise api.TirError(kind, msg)


def tensorize(ir: str, block: str):
    L = adapter()
    text = ctypes.create_string_buffer(1 << 20)
    trace = ctypes.create_string_buffer(1 << 16)
    intrin = ctypes.create_string_buffer(256)
    desc = api.ConvDesc()
    mnk = (ctypes.c_int64 * 3)()
    err = ctypes.create_string_buffer(2048)
    rc = L.tir_b200_adapter_tensorize(ir.encode(), block.encode(), text, len(text), trace, len(trace), intrin,
                                      len(intrin), ctypes.byref(desc), mnk, err, len(err))
    if rc != 0:
        _raise(err)
    return text.value.decode(), trace.value.decode(), intrin.value.decode(), desc, tuple(mnk)


def run_auto(ir: str, blocks, inputs, out_shape):
    L = adapter()
    ins = [np.ascontiguousarray(x, np.float32) for x in inputs]
    f32p = ctypes.POINTER(ctypes.c_float)
    arr = (f32p * len(ins))(*[x.ctypes.data_as(f32p) for x in ins])
    names = (ctypes.c_char_p * len(blocks))(*[b.encode() for b in blocks])
    out = np.zeros(out_shape, np.float32)
    calls = ctypes.c_int64(0)
    err = ctypes.create_string_buffer(2048)
    rc = L.tir_b200_adapter_run_auto(ir.encode(), names, len(blocks), len(ins), arr, out.ctypes.data_as(f32p),
                                     out.size, ctypes.byref(calls), err, len(err))
    if rc != 0:
        _raise(err)
    return out, calls.value


def ref_workload(which, *args):
    lib = O._ref()
    lib.tirref_workload_source.restype = ctypes.c_char_p
    lib.tirref_workload_source.argtypes = [ctypes.c_char_p] + [ctypes.c_int] * 6
    args = list(args) + [0] * (6 - len(args))
    return lib.tirref_workload_source(which.encode(), *args).decode()


SPECS = {
    "C1D": G.ConvSpec("C1D", n=2, in_dhw=(1, 1, 10), ci=8, co=16, k=(1, 1, 3), s=(1, 1, 2), p=(0, 0, 1)),
    "C2D": G.ConvSpec("C2D", n=2, in_dhw=(1, 7, 6), ci=8, co=16, k=(1, 3, 3), p=(0, 1, 1)),
    "C2D_nopad": G.ConvSpec("C2D", n=1, in_dhw=(1, 6, 6), ci=16, co=8, k=(1, 3, 3)),
    "C3D": G.ConvSpec("C3D", n=1, in_dhw=(4, 5, 5), ci=3, co=8, k=(3, 3, 3), s=(2, 2, 2), p=(1, 1, 1)),
    "DIL": G.ConvSpec("DIL", n=1, in_dhw=(1, 11, 11), ci=3, co=8, k=(1, 3, 3), s=(1, 2, 2), p=(0, 2, 2), d=(1, 2, 2)),
    "GRP": G.ConvSpec("GRP", n=1, in_dhw=(1, 6, 6), ci=16, co=32, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=4),
    "T2D": G.ConvSpec("T2D", n=2, in_dhw=(1, 3, 3), ci=8, co=8, k=(1, 4, 4), s=(1, 2, 2), p=(0, 1, 1), transposed=True),
    "T2D_s1": G.ConvSpec("T2D", n=1, in_dhw=(1, 4, 4), ci=8, co=8, k=(1, 3, 3), s=(1, 1, 1), p=(0, 1, 1), transposed=True),
    "DEP": G.ConvSpec("DEP", n=2, in_dhw=(1, 6, 6), ci=8, co=8, k=(1, 3, 3), p=(0, 1, 1), groups=8),
    "DEP_s2": G.ConvSpec("DEP", n=1, in_dhw=(1, 9, 9), ci=16, co=16, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=16),
}


def _check_desc(d, spec: G.ConvSpec):
    assert d.op == OPS[spec.op]
    assert d.transposed == int(spec.transposed)
    assert (d.n, d.ci, d.co, d.groups) == (spec.n, spec.ci, spec.co, spec.groups)
    assert (d.in_d, d.in_h, d.in_w) == tuple(spec.in_dhw)
    assert (d.k_d, d.k_h, d.k_w) == tuple(spec.k)
    assert (d.s_d, d.s_h, d.s_w) == tuple(spec.s)
    assert (d.p_d, d.p_h, d.p_w) == tuple(spec.p)
    assert (d.d_d, d.d_h, d.d_w) == tuple(spec.d)


@pytest.mark.parametrize("name", list(SPECS))
def test_match_recovers_conv_geometry(name):
    spec = SPECS[name]
    text, trace, intrin, d, _ = tensorize(G.conv_source(spec), "conv")
    _check_desc(d, spec)
    assert f'attrs("tensorized" = "{intrin}")' in text
    assert f"{intrin}()" in text
    assert "block conv(" not in text  # the scalar inner block is gone
    assert [line.split('"prim":"')[1].split('"')[0] for line in trace.splitlines()] == ["blockize", "b200.tensorize"]


def test_match_gmm_and_reference_workloads():
    text, _, intrin, d, mnk = tensorize(G.gmm_source(24, 40, 56), "gemm")
    assert d.op == OPS["GMM"] and mnk == (24, 40, 56) and intrin == "b200.gmm.ow"
    # the reference's own programs (tests/testing/workloads.h), f32 params
    _, _, intrin, d, mnk = tensorize(ref_workload("matmul", 16), "gemm")
    assert intrin == "b200.gmm.ow" and mnk == (16, 16, 16)
    _, _, _, d, _ = tensorize(ref_workload("conv2d", 8, 8, 4, 3, 3, 8), "conv")
    _check_desc(d, G.ConvSpec("C2D", n=1, in_dhw=(1, 8, 8), ci=4, co=8, k=(1, 3, 3)))
    _, _, _, d, _ = tensorize(ref_workload("depthwise", 8, 8, 8, 3, 3), "dw")
    _check_desc(d, G.ConvSpec("DEP", n=1, in_dhw=(1, 8, 8), ci=8, co=8, k=(1, 3, 3), groups=8))
    # gemm_relu: only the gemm block is a contraction
    text, _, _, _, mnk = tensorize(ref_workload("gemm_relu", 16), "gemm")
    assert mnk == (16, 16, 16) and "block relu(" in text


def test_rejects_non_contractions_and_partial_nests():
    with pytest.raises(api.TirError) as e:
        tensorize(ref_workload("gemm_relu", 8), "relu")
    assert e.value.kind == "DescMismatch"
    with pytest.raises(api.TirError) as e:  # a row slice covers part of the op
        tensorize(G.gmm_source(32, 16, 16, rows=(0, 16)), "gemm")
    assert e.value.kind in ("DescMismatch", "NotWholeOp", "NotSeparable")
    with pytest.raises(api.TirError) as e:
        tensorize(G.conv_source(SPECS["C2D"], rows=(2, 5)), "conv")
    assert e.value.kind in ("DescMismatch", "NotWholeOp", "NotSeparable")
    with pytest.raises(api.TirError) as e:
        tensorize(G.gmm_source(16, 16, 16), "nope")
    assert e.value.kind == "StaleHandle"
    # a padded conv whose guard was dropped would read out of bounds
    unguarded = re.sub(r"select\((.*?), (f32\(A\[[^\]]*\]\)), 0\.0\)", r"\2", G.conv_source(SPECS["C2D"]))
    assert "select(" not in unguarded
    with pytest.raises(api.TirError) as e:
        tensorize(unguarded, "conv")
    assert e.value.kind == "DescMismatch"
    # a guarded (predicated) contraction writes part of its domain: never whole-op
    guarded = G.gmm_source(16, 16, 16).replace(") {\n            init", ") if i < 8 {\n            init")
    assert " if i < 8 {" in guarded
    with pytest.raises(api.TirError) as e:
        tensorize(guarded, "gemm")
    assert e.value.kind == "DescMismatch" and "predicate" in e.value.message


def test_tensorized_block_init_and_regions():
    """blockize moves the zero init to the outer block (schedule_block.cc:570-603);
    for a whole-op block it would run once, right before the single call, so the
    composite folds it into an overwriting intrinsic ('.ow': Y = op(X, W), the
    output is neither zero-filled by the interpreter nor uploaded). A block
    WITHOUT init (accumulate into Y) keeps the accumulating intrinsic."""
    text, trace, intrin, _, _ = tensorize(G.conv_source(SPECS["GRP"]), "conv")
    assert "init {" not in text and intrin.endswith(".ow") and '"drop_init":true' in trace.replace(" ", "")
    assert text.count("tensorized") == 1 and "reads(" in text and "writes(" in text
    no_init = re.sub(r"init \{[^}]*\}\s*", "", G.conv_source(SPECS["GRP"]))
    assert "init {" not in no_init
    text2, _, intrin2, _, _ = tensorize(no_init, "conv")
    assert not intrin2.endswith(".ow") and intrin2 + ".ow" == intrin


# ---------------------------------------------------------------- GPU: run it


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(SPECS))
def test_tensorized_program_runs_on_b200_bit_exact(name, cuda):
    spec = SPECS[name]
    x = O.reference_tensor(spec.x_shape(), 1)
    w = O.reference_tensor(spec.w_shape(), 2)
    out, calls = run_auto(G.conv_source(spec), ["conv"], [x, w], spec.y_shape())
    assert calls == 1
    assert O.tensors_bitwise_equal(out, O.conv(spec, x, w))


@pytest.mark.gpu
def test_reference_gemm_relu_program_tensorized(golden, cuda):
    meta, arrays = golden
    a, b, want = arrays["ref_gemm_relu16/a"], arrays["ref_gemm_relu16/b"], arrays["ref_gemm_relu16/out"]
    out, calls = run_auto(ref_workload("gemm_relu", 16), ["gemm"], [a, b], (16, 16))
    assert calls == 1
    assert O.tensors_bitwise_equal(out, want)


@pytest.mark.gpu
def test_epilogue_program_with_tensorized_conv(cuda):
    spec = G.ConvSpec("C2D", n=2, in_dhw=(1, 9, 9), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1))
    x = O.reference_tensor(spec.x_shape(), 3)
    w = O.reference_tensor(spec.w_shape(), 4)
    bias = O.reference_tensor((spec.co,), 5)
    src = G.with_epilogue(G.conv_source(spec), spec.y_shape(), bias=True, relu=True)
    out, calls = run_auto(src, ["conv"], [x, w, bias], spec.y_shape())
    assert calls == 1
    assert O.tensors_bitwise_equal(out, O.epilogue(O.conv(spec, x, w), bias, True))


def declare(ir: str, block: str) -> str:
    L = adapter()
    L.tir_b200_adapter_declare.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int64,
                                           ctypes.c_char_p, ctypes.c_int]
    out = ctypes.create_string_buffer(1 << 20)
    err = ctypes.create_string_buffer(2048)
    if L.tir_b200_adapter_declare(ir.encode(), block.encode(), out, len(out), err, len(err)) != 0:
        _raise(err)
    return out.value.decode()


def run_declared(program: str, inputs, out_shape):
    L = adapter()
    f32p = ctypes.POINTER(ctypes.c_float)
    L.tir_b200_adapter_run_declared.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(f32p), f32p,
                                                ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), ctypes.c_char_p,
                                                ctypes.c_int]
    ins = [np.ascontiguousarray(x, np.float32) for x in inputs]
    arr = (f32p * len(ins))(*[x.ctypes.data_as(f32p) for x in ins])
    out = np.zeros(out_shape, np.float32)
    calls = ctypes.c_int64(0)
    err = ctypes.create_string_buffer(2048)
    if L.tir_b200_adapter_run_declared(program.encode(), len(ins), arr, out.ctypes.data_as(f32p), out.size,
                                       ctypes.byref(calls), err, len(err)) != 0:
        _raise(err)
    return out, calls.value


@pytest.mark.parametrize("name", ["C2D", "T2D", "DEP", "C3D"])
def test_intrin_declaration_round_trips(name):
    """the tensorized program carries an `intrin` declaration
    of its B200 intrinsic in the reference grammar (parser.cc:749-781): one
    `require <view> scope("global") contiguous` per view ([writes[0], reads...]),
    no exec_scope; it parses back with tir::parse_program (checked inside)."""
    prog = declare(G.conv_source(SPECS[name]), "conv")
    head = prog.split("\n\n")[0]
    assert head.startswith("intrin b200.") and ".ow {" in head
    assert head.count('scope("global") contiguous') == 3 and "exec_scope" not in head
    assert "func " in prog and "tensorized" in prog


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C2D", "GRP", "T2D", "DEP"])
def test_registry_from_declarations_runs_bit_exact(name, cuda):
    """The kernel registry built from the program's own declarations
    (register_declared decodes the full geometry from the intrinsic name):
    tir::run of the declared program is bit-exact vs the oracle."""
    spec = SPECS[name]
    x = O.reference_tensor(spec.x_shape(), 1)
    w = O.reference_tensor(spec.w_shape(), 2)
    out, calls = run_declared(declare(G.conv_source(spec), "conv"), [x, w], spec.y_shape())
    assert calls == 1
    assert O.tensors_bitwise_equal(out, O.conv(spec, x, w))


def test_declarations_reject_foreign_requirements():
    prog = declare(G.conv_source(SPECS["C2D"]), "conv")
    bad = prog.replace('scope("global")', 'scope("shared")', 1)
    with pytest.raises(api.TirError) as e:
        run_declared(bad, [np.zeros(SPECS["C2D"].x_shape(), np.float32),
                           np.zeros(SPECS["C2D"].w_shape(), np.float32)], SPECS["C2D"].y_shape())
    assert e.value.kind == "DescMismatch"
