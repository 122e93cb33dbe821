"""Generates tests/golden/golden.npz from the REFERENCE interpreter.

Run in the build container (needs /root/reference and oracle/_ref built):
    python tests/golden/make_golden.py

Every output here is produced by tir::run (/root/reference/proj/src/interp.cc:579)
via oracle/_ref/libtirref.so, on inputs from the reference's own seeded
generator random_tensor (tests/testing/workloads.h:170-184, called through the
shim so the fixture does not depend on our Python mt19937_64 port):
  * the reference's own workload programs exactly as its tests run them
    (matmul_source, conv2d_source, depthwise_source; tests/test_interp.cc:29-73);
  * our reference-grammar programs (oracle/ir_gen.py) for every op of the
    paper's set, with batch / stride / padding / dilation / groups / transposed;
  * one fp16-rounded-normal (D2) case per op family.
The fixture is small (a few hundred KB) and is what `-m "not gpu"` tests pin
the C restatement (oracle/tir_oracle.c) against.
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

CASES = {
    "C1D": G.ConvSpec("C1D", n=2, in_dhw=(1, 1, 10), ci=8, co=16, k=(1, 1, 3), s=(1, 1, 2), p=(0, 0, 1)),
    "C2D": G.ConvSpec("C2D", n=2, in_dhw=(1, 7, 6), ci=8, co=16, k=(1, 3, 3), p=(0, 1, 1)),
    "C2D_s2": G.ConvSpec("C2D", n=1, in_dhw=(1, 9, 9), ci=16, co=8, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1)),
    "C3D": G.ConvSpec("C3D", n=1, in_dhw=(4, 5, 5), ci=3, co=8, k=(3, 3, 3), s=(2, 2, 2), p=(1, 1, 1)),
    "DIL": G.ConvSpec("DIL", n=1, in_dhw=(1, 11, 11), ci=3, co=8, k=(1, 3, 3), s=(1, 2, 2), p=(0, 2, 2), d=(1, 2, 2)),
    "GRP": G.ConvSpec("GRP", n=1, in_dhw=(1, 6, 6), ci=16, co=32, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=4),
    "T2D": G.ConvSpec("T2D", n=2, in_dhw=(1, 3, 3), ci=8, co=8, k=(1, 4, 4), s=(1, 2, 2), p=(0, 1, 1), transposed=True),
    "DEP": G.ConvSpec("DEP", n=2, in_dhw=(1, 6, 6), ci=8, co=8, k=(1, 3, 3), p=(0, 1, 1), groups=8),
    "DEP_s2": G.ConvSpec("DEP", n=1, in_dhw=(1, 9, 9), ci=16, co=16, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=16),
}
GMM_CASES = {"GMM_16": (16, 16, 16), "GMM_24x40x56": (24, 40, 56)}


def ref_tensor(lib, shape, seed):
    n = int(np.prod(shape))
    out = np.zeros(n, np.float32)
    assert lib.tirref_random_tensor(n, seed, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float))) == 0
    return out.reshape(shape)


def main():
    lib = O._ref()
    lib.tirref_random_tensor.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_float)]
    lib.tirref_workload_source.restype = ctypes.c_char_p
    lib.tirref_workload_source.argtypes = [ctypes.c_char_p] + [ctypes.c_int] * 6
    arrays, meta = {}, {}

    # 1. the reference's own programs, as tests/test_interp.cc:29-73 runs them
    own = {
        "ref_matmul16": (("matmul", 16, 0, 0, 0, 0, 0), [(16, 16), (16, 16)], (1, 2), (16, 16)),
        "ref_conv2d": (("conv2d", 8, 8, 4, 3, 3, 8), [(1, 8, 8, 4), (3, 3, 4, 8)], (7, 8), (1, 6, 6, 8)),
        "ref_depthwise": (("depthwise", 8, 8, 8, 3, 3, 0), [(1, 8, 8, 8), (3, 3, 8)], (9, 10), (1, 6, 6, 8)),
    }
    for name, (src_args, shapes, seeds, out_shape) in own.items():
        src = lib.tirref_workload_source(src_args[0].encode(), *src_args[1:]).decode()
        ins = [ref_tensor(lib, s, sd) for s, sd in zip(shapes, seeds)]
        out, _ = O.ref_run(src, ins, out_shape)
        arrays[f"{name}/a"], arrays[f"{name}/b"], arrays[f"{name}/out"] = ins[0], ins[1], out
        meta[name] = {"kind": "reference_workload", "source": list(src_args), "seeds": list(seeds)}

    # 2. our reference-grammar programs for the paper's op set (D1)
    for name, (m, n, k) in GMM_CASES.items():
        a = ref_tensor(lib, (m, k), 1)
        b = ref_tensor(lib, (k, n), 2)
        out, _ = O.ref_run(G.gmm_source(m, n, k), [a, b], (m, n))
        arrays[f"{name}/a"], arrays[f"{name}/b"], arrays[f"{name}/out"] = a, b, out
        meta[name] = {"kind": "gmm", "mnk": [m, n, k], "dist": "D1"}
    for name, spec in CASES.items():
        x = ref_tensor(lib, spec.x_shape(), 3)
        w = ref_tensor(lib, spec.w_shape(), 4)
        out, _ = O.ref_run(G.conv_source(spec), [x, w], spec.y_shape())
        arrays[f"{name}/a"], arrays[f"{name}/b"], arrays[f"{name}/out"] = x, w, out
        meta[name] = {"kind": "conv", "spec": spec.__dict__, "dist": "D1"}

    # 3. D2: fp16-rounded normals
    for name in ["C2D", "GRP", "T2D", "DEP"]:
        spec = CASES[name]
        x = O.normal_f16(spec.x_shape(), 11)
        w = O.normal_f16(spec.w_shape(), 12)
        out, _ = O.ref_run(G.conv_source(spec), [x, w], spec.y_shape())
        key = f"{name}_D2"
        arrays[f"{key}/a"], arrays[f"{key}/b"], arrays[f"{key}/out"] = x, w, out
        meta[key] = {"kind": "conv", "spec": spec.__dict__, "dist": "D2"}

    # 4. fused epilogues: the reference's own gemm_relu
    # program (f32 params; random_tensor values are fp16-exact), then bias/relu
    # stages appended to our programs by ir_gen.with_epilogue.
    src = lib.tirref_workload_source(b"gemm_relu", 16, 0, 0, 0, 0, 0).decode()
    ins = [ref_tensor(lib, (16, 16), 1), ref_tensor(lib, (16, 16), 2)]
    out, _ = O.ref_run(src, ins, (16, 16))
    arrays["ref_gemm_relu16/a"], arrays["ref_gemm_relu16/b"], arrays["ref_gemm_relu16/out"] = *ins, out
    meta["ref_gemm_relu16"] = {"kind": "reference_workload", "source": ["gemm_relu", 16, 0, 0, 0, 0, 0],
                               "seeds": [1, 2], "epilogue": {"bias": False, "relu": True}}
    for name, base, bias, relu in [("GMM_24x40x56_bias_relu", "GMM_24x40x56", True, True),
                                   ("C2D_bias_relu", "C2D", True, True), ("GRP_bias", "GRP", True, False),
                                   ("T2D_relu", "T2D", False, True), ("DEP_bias_relu", "DEP", True, True)]:
        a, b = arrays[f"{base}/a"], arrays[f"{base}/b"]
        if base.startswith("GMM"):
            m, n, k = GMM_CASES[base]
            body, out_shape, m_ = G.gmm_source(m, n, k), (m, n), {"kind": "gmm", "mnk": [m, n, k]}
        else:
            spec = CASES[base]
            body, out_shape, m_ = G.conv_source(spec), spec.y_shape(), {"kind": "conv", "spec": spec.__dict__}
        ins = [a, b]
        if bias:
            ins.append(ref_tensor(lib, (out_shape[-1],), 5))
            arrays[f"{name}/bias"] = ins[-1]
        out, _ = O.ref_run(G.with_epilogue(body, out_shape, bias, relu), ins, out_shape)
        arrays[f"{name}/a"], arrays[f"{name}/b"], arrays[f"{name}/out"] = a, b, out
        meta[name] = {**m_, "dist": "D1", "epilogue": {"bias": bias, "relu": relu}}

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, default=list)
    print(f"wrote {len(meta)} cases")


if __name__ == "__main__":
    main()
