"""The reference's tensor-file format — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Restates read_tensor / write_tensor (/root/reference/proj/src/interp.cc:730-769):
a text header line `dtype d0 d1 ...\\n` followed by the raw little-endian
elements; F16 tensors are stored with 4-byte f32 elements (the interpreter's F16
is an f32 tag, src/ir.cc:36-47). Used to read the on-disk golden vectors in
tests/golden/ref_format/ on machines without the reference (the GPU box).
"""
from __future__ import annotations

import numpy as np

_DT = {"f32": np.float32, "f16": np.float32, "i32": np.int32, "i8": np.int8}


def read_tensor(path: str) -> tuple[str, np.ndarray]:
    with open(path, "rb") as f:
        header = f.readline().decode().split()
        dtype, shape = header[0], tuple(int(d) for d in header[1:])
        if dtype not in _DT:
            raise ValueError(f"bad tensor header in '{path}'")
        data = np.frombuffer(f.read(), dtype=_DT[dtype])
    n = int(np.prod(shape)) if shape else 1
    if data.size < n:
        raise ValueError(f"tensor file '{path}' is truncated")
    return dtype, data[:n].reshape(shape).copy()


def write_tensor(path: str, dtype: str, arr: np.ndarray) -> None:
    with open(path, "wb") as f:
        f.write((" ".join([dtype] + [str(d) for d in arr.shape]) + "\n").encode())
        f.write(np.ascontiguousarray(arr, _DT[dtype]).tobytes())
