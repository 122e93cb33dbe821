"""the channel pad of small-CI convolutions as IR steps of
the reference's own schedule API instead of a device relayout.

adapter/tir_b200_tensorize.cc::pad_conv_channels stages X and W
(Schedule::cache_read, schedule_block.cc:283), grows the channel reduction to a
multiple of 8 (Schedule::pad_block, schedule_block.cc:1186; the staged copies
are zero-filled by the guarded producers pad_block emits) and widens the conv's
declared read regions to whole buffers (a recorded, replayable
"b200.widen_reads" step). CPU: tir::run of the padded program equals the
original bit for bit, the trace holds the reference's own steps and replays.
GPU: the padded program's conv block tensorizes onto b200.conv with CI = 8 —
the kernel sees 16-byte pixel rows without the device pad — while the two
staging blocks stay scalar in the interpreter; the result is bit-exact.
"""
import ctypes
import json
import os

import numpy as np
import pytest

from oracle import ir_gen as G
from oracle import oracle as O
from paper_2207_04296_b200 import api

ADAPTER = os.path.join(os.path.dirname(api.LIB_PATH), "libtir_b200_adapter.so")
CASES = {
    "DIL": G.ConvSpec("DIL", n=1, in_dhw=(1, 12, 12), ci=3, co=16, k=(1, 3, 3), s=(1, 2, 2), p=(0, 2, 2), d=(1, 2, 2)),
    "C2D_stem": G.ConvSpec("C2D", n=2, in_dhw=(1, 9, 9), ci=3, co=8, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1)),
    "C3D": G.ConvSpec("C3D", n=1, in_dhw=(3, 5, 5), ci=3, co=8, k=(3, 3, 3), s=(2, 2, 2), p=(1, 1, 1)),
    "C1D": G.ConvSpec("C1D", n=2, in_dhw=(1, 1, 11), ci=5, co=8, k=(1, 1, 3), p=(0, 0, 1)),
}


def adapter():
    if not os.path.exists(ADAPTER):
        pytest.skip("adapter library not built (needs /root/reference at build time)")
    L = ctypes.CDLL(ADAPTER)
    L.tir_b200_adapter_pad_channels.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p,
                                                ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64,
                                                ctypes.POINTER(ctypes.c_int64), ctypes.c_char_p, ctypes.c_int]
    return L


def pad(src: str):
    L = adapter()
    text = ctypes.create_string_buffer(1 << 20)
    trace = ctypes.create_string_buffer(1 << 16)
    err = ctypes.create_string_buffer(1024)
    padded = ctypes.c_int64()
    rc = L.tir_b200_adapter_pad_channels(src.encode(), b"conv", 8, text, len(text), trace, len(trace),
                                         ctypes.byref(padded), err, len(err))
    if rc != 0:
        kind, _, msg = err.value.decode().partition("|")
        raise api.TirError(kind, msg)
    return text.value.decode(), trace.value.decode(), padded.value


@pytest.mark.parametrize("name", sorted(CASES))
def test_channel_pad_as_ir_steps_is_exact(name):
    if not O.ref_available():
        pytest.skip("reference interpreter not built here")
    spec = CASES[name]
    src = G.conv_source_direct(spec)
    text, trace, padded = pad(src)
    assert padded == 8
    steps = [json.loads(ln)["prim"] for ln in trace.strip().splitlines()]
    assert steps == ["cache_read", "cache_read", "pad_block", "b200.widen_reads"]
    assert "select(" in text and f"0..{padded}" in text
    x = O.reference_tensor(spec.x_shape(), 1)
    w = O.reference_tensor(spec.w_shape(), 2)
    want, _ = O.ref_run(src, [x, w], spec.y_shape())
    got, _ = O.ref_run(text, [x, w], spec.y_shape())
    assert O.tensors_bitwise_equal(got, want)
    assert O.tensors_bitwise_equal(want, O.conv(spec, x, w))


def test_pad_rejects_non_conv_block():
    with pytest.raises(api.TirError) as e:
        pad(G.gmm_source(16, 16, 16).replace("block gemm", "block conv"))
    assert e.value.kind == "DescMismatch"


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_padded_program_tensorizes_onto_b200(name, cuda):
    from test_tensorize import run_auto  # tests/ is on sys.path (pytest prepend import mode)

    spec = CASES[name]
    text, _, _ = pad(G.conv_source_direct(spec))
    x = O.reference_tensor(spec.x_shape(), 3)
    w = O.reference_tensor(spec.w_shape(), 4)
    got, calls = run_auto(text, ["conv"], [x, w], spec.y_shape())
    assert calls == 1
    assert O.tensors_bitwise_equal(got, O.conv(spec, x, w))
