"""Golden vectors in the reference's own tensor-file format.

tests/golden/ref_format/<case>/{in0,in1,out}.tensor were written by
tir::write_tensor from tir::run outputs (tests/golden/make_ref_tensors.py). CPU
tests: our reader (oracle/tensor_file.py) agrees with the reference's own
read_tensor (src/interp.cc:730-759) where the reference is built, and the C
restatement reproduces every golden output bit for bit. GPU tests: the CUDA
kernels, fed the golden inputs through the device C-ABI, reproduce the golden
outputs bit for bit (reference input distribution, exact partial sums).
"""
import ctypes
import json
import os

import numpy as np
import pytest

from oracle import ir_gen as G
from oracle import oracle as O
from oracle import tensor_file as TF

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_format")
MANIFEST = json.load(open(os.path.join(HERE, "manifest.json")))


def load(name):
    _, x = TF.read_tensor(os.path.join(HERE, name, "in0.tensor"))
    _, w = TF.read_tensor(os.path.join(HERE, name, "in1.tensor"))
    _, y = TF.read_tensor(os.path.join(HERE, name, "out.tensor"))
    return x, w, y


def spec_of(meta):
    return G.ConvSpec(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in meta.items()})


@pytest.mark.parametrize("name", sorted(MANIFEST))
def test_reader_matches_reference_read_tensor(name):
    if not O.ref_available():
        pytest.skip("reference interpreter not built here")
    lib = O._ref()
    lib.tirref_read_tensor.restype = ctypes.c_int64
    lib.tirref_read_tensor.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_float), ctypes.c_int64,
                                       ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]
    for f in ("in0", "in1", "out"):
        path = os.path.join(HERE, name, f + ".tensor")
        dtype, ours = TF.read_tensor(path)
        shape = (ctypes.c_int64 * 8)()
        nd = ctypes.c_int()
        buf = np.zeros(ours.size, np.float32)
        n = lib.tirref_read_tensor(path.encode(), buf.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), buf.size,
                                   shape, ctypes.byref(nd))
        assert n == ours.size and tuple(shape[:nd.value]) == ours.shape
        assert np.array_equal(buf.reshape(ours.shape), ours)
        assert dtype == ("f32" if f == "out" else "f16")


def test_writer_round_trip(tmp_path):
    a = np.arange(24, dtype=np.float32).reshape(2, 3, 4) / 8
    p = str(tmp_path / "t.tensor")
    TF.write_tensor(p, "f16", a)
    dtype, b = TF.read_tensor(p)
    assert dtype == "f16" and np.array_equal(a, b)
    assert open(p, "rb").readline() == b"f16 2 3 4\n"


@pytest.mark.parametrize("name", sorted(MANIFEST))
def test_restatement_reproduces_golden(name):
    x, w, y = load(name)
    meta = MANIFEST[name]
    got = O.gmm(x, w) if meta["op"] == "GMM" else O.conv(spec_of(meta), x, w)
    assert O.tensors_bitwise_equal(got, y)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(MANIFEST))
def test_cuda_reproduces_golden(name, cuda):
    import torch

    import paper_2207_04296_b200 as tb

    x, w, y = load(name)
    meta = MANIFEST[name]
    X = torch.from_numpy(x).to(cuda).half()
    W = torch.from_numpy(w).to(cuda).half()
    if meta["op"] == "GMM":
        got = tb.gmm(X, W)
    else:
        s = spec_of(meta)
        spec = tb.Conv(s.op, n=s.n, in_dhw=s.in_dhw, ci=s.ci, co=s.co, k=s.k, s=s.s, p=s.p, d=s.d, groups=s.groups,
                       transposed=s.transposed)
        got = tb.conv(spec, X, W)
    torch.cuda.synchronize()
    assert O.tensors_bitwise_equal(got.cpu().numpy(), y)
