"""Writes tests/golden/ref_format/: golden vectors in the REFERENCE's own tensor-file
format, produced end to end by the reference.

Run in the build container (needs /root/reference and oracle/_ref built):
    python tests/golden/make_ref_tensors.py

For every case the inputs come from the reference's seeded generator
random_tensor (tests/testing/workloads.h:170-184, through the shim), are written
with tir::write_tensor (src/interp.cc:761-769) as F16 tensors, and the output is
tir::run (interp.cc:579) of the op's reference-grammar program over the inputs
read back with tir::read_tensor (interp.cc:730-759), written with write_tensor.
The files travel to the GPU box, where tests read them with oracle/tensor_file.py.
"""
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ir_gen as G  # noqa: E402
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(HERE, "ref_format")
CASES = {
    "C1D": G.ConvSpec("C1D", n=2, in_dhw=(1, 1, 20), ci=16, co=32, k=(1, 1, 3), s=(1, 1, 2), p=(0, 0, 1)),
    "C2D": G.ConvSpec("C2D", n=2, in_dhw=(1, 10, 10), ci=64, co=32, k=(1, 3, 3), p=(0, 1, 1)),
    "C3D": G.ConvSpec("C3D", n=1, in_dhw=(4, 6, 6), ci=3, co=16, k=(3, 3, 3), s=(2, 2, 2), p=(1, 1, 1)),
    "DIL": G.ConvSpec("DIL", n=1, in_dhw=(1, 12, 12), ci=3, co=16, k=(1, 3, 3), s=(1, 2, 2), p=(0, 2, 2), d=(1, 2, 2)),
    "GRP": G.ConvSpec("GRP", n=1, in_dhw=(1, 8, 8), ci=32, co=64, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=4),
    "T2D": G.ConvSpec("T2D", n=2, in_dhw=(1, 3, 3), ci=32, co=16, k=(1, 4, 4), s=(1, 2, 2), p=(0, 1, 1),
                      transposed=True),
    "DEP": G.ConvSpec("DEP", n=2, in_dhw=(1, 9, 9), ci=32, co=32, k=(1, 3, 3), p=(0, 1, 1), groups=32),
}
GMM = {"GMM": (64, 48, 80)}  # M, N, K


def main():
    lib = O._ref()
    f32p = ctypes.POINTER(ctypes.c_float)
    lib.tirref_random_tensor.argtypes = [ctypes.c_int64, ctypes.c_uint64, f32p]
    lib.tirref_write_tensor.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int64), f32p]
    lib.tirref_run_files.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_char_p), ctypes.c_char_p]
    lib.tirref_last_error.restype = ctypes.c_char_p

    def check(rc):
        if rc != 0:
            raise RuntimeError(lib.tirref_last_error().decode())

    def write_input(path, shape, seed):
        n = int(np.prod(shape))
        buf = np.zeros(n, np.float32)
        check(lib.tirref_random_tensor(n, seed, buf.ctypes.data_as(f32p)))
        dims = (ctypes.c_int64 * len(shape))(*shape)
        check(lib.tirref_write_tensor(path.encode(), b"f16", len(shape), dims, buf.ctypes.data_as(f32p)))

    os.makedirs(OUT, exist_ok=True)
    manifest = {}
    progs = {}
    for name, (m, n, k) in GMM.items():
        progs[name] = (G.gmm_source(m, n, k), [(m, k), (k, n)], {"op": "GMM", "mnk": [m, n, k]})
    for name, spec in CASES.items():
        meta = {f: getattr(spec, f) for f in ("op", "n", "in_dhw", "ci", "co", "k", "s", "p", "d", "groups",
                                              "transposed")}
        progs[name] = (G.conv_source(spec), [spec.x_shape(), spec.w_shape()], meta)
    for seed_base, (name, (text, shapes, meta)) in enumerate(sorted(progs.items())):
        d = os.path.join(OUT, name)
        os.makedirs(d, exist_ok=True)
        ins = []
        for i, shape in enumerate(shapes):
            path = os.path.join(d, f"in{i}.tensor")
            write_input(path, tuple(int(s) for s in shape), 1000 * (seed_base + 1) + i)
            ins.append(path.encode())
        arr = (ctypes.c_char_p * len(ins))(*ins)
        check(lib.tirref_run_files(text.encode(), len(ins), arr, os.path.join(d, "out.tensor").encode()))
        manifest[name] = meta
        print(name, "ok")
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, default=list)


if __name__ == "__main__":
    main()
