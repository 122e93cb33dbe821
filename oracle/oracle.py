"""ctypes front-end of the oracle — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl
reference legs import this module, and only as the checker or the timed CPU
reference. It wraps
  * oracle/lib/libtir_oracle.so — our plain-C restatement (tir_oracle.c);
  * oracle/_ref/libtirref.so    — the reference interpreter itself
    (tir::run over /root/reference/proj/src, built by oracle/Makefile).
Also: the reference's seeded input distribution (random_tensor,
/root/reference/proj/tests/testing/workloads.h:170-184) and its comparators
(tensors_close :264-282, tensors_bitwise_equal :284-298).
"""
from __future__ import annotations

import ctypes
import os
import time

import numpy as np

from .ir_gen import ConvSpec

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "lib", "libtir_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libtirref.so")

_OP_CODES = {"GMM": 0, "C1D": 1, "C2D": 2, "C3D": 3, "DIL": 4, "GRP": 5, "T2D": 6, "DEP": 7}


class ConvDesc(ctypes.Structure):
    """Mirror of tir_b200_conv_desc (include/tir_b200.h)."""

    _fields_ = [
        ("op", ctypes.c_int32), ("transposed", ctypes.c_int32), ("n", ctypes.c_int64),
        ("in_d", ctypes.c_int64), ("in_h", ctypes.c_int64), ("in_w", ctypes.c_int64),
        ("ci", ctypes.c_int64), ("co", ctypes.c_int64),
        ("k_d", ctypes.c_int64), ("k_h", ctypes.c_int64), ("k_w", ctypes.c_int64),
        ("s_d", ctypes.c_int64), ("s_h", ctypes.c_int64), ("s_w", ctypes.c_int64),
        ("p_d", ctypes.c_int64), ("p_h", ctypes.c_int64), ("p_w", ctypes.c_int64),
        ("d_d", ctypes.c_int64), ("d_h", ctypes.c_int64), ("d_w", ctypes.c_int64),
        ("groups", ctypes.c_int64),
    ]

    @classmethod
    def from_spec(cls, s: ConvSpec) -> "ConvDesc":
        return cls(_OP_CODES[s.op], int(s.transposed), s.n, *s.in_dhw, s.ci, s.co, *s.k, *s.s,
                   *s.p, *s.d, s.groups)


# ---------------- inputs (workloads.h:170-184) ----------------

class _MT19937_64:
    """std::mt19937_64 (the reference seeds one generator per operand)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.idx = 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) + (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def next(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEB5A0000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def _mt_stream_mod64(seed: int, count: int) -> np.ndarray:
    """rng() % 64 for `count` draws of std::mt19937_64(seed), vectorised twist."""
    mt = np.zeros(312, dtype=np.uint64)
    gen = _MT19937_64(seed)
    mt[:] = np.array(gen.mt, dtype=np.uint64)
    out = np.empty(count, dtype=np.uint64)
    pos = 0
    U, L = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)
    A = np.uint64(0xB5026F5AA96619E9)
    while pos < count:
        # twist (sequential dependency within blocks of 156; do it in 3 slices)
        for lo, hi in ((0, 156), (156, 311), (311, 312)):
            i = np.arange(lo, hi)
            x = (mt[i] & U) | (mt[(i + 1) % 312] & L)
            xa = x >> np.uint64(1)
            xa = np.where((x & np.uint64(1)) != 0, xa ^ A, xa)
            mt[i] = mt[(i + 156) % 312] ^ xa
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEB5A0000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        take = min(312, count - pos)
        out[pos:pos + take] = y[:take]
        pos += take
    return (out % np.uint64(64)).astype(np.int64)


def reference_tensor(shape, seed: int) -> np.ndarray:
    """random_tensor(F32/F16, shape, seed): (rng() % 64) / 8 - 4 (workloads.h:176)."""
    count = int(np.prod(shape)) if len(shape) else 1
    k = _mt_stream_mod64(seed, count)
    return (k.astype(np.float32) / np.float32(8.0) - np.float32(4.0)).reshape(shape)


def normal_f16(shape, seed: int) -> np.ndarray:
    """D2: N(0,1) rounded to fp16 (RN), returned as f32 values."""
    rng = np.random.Generator(np.random.MT19937(seed))
    return rng.standard_normal(size=shape, dtype=np.float32).astype(np.float16).astype(np.float32)


# ---------------- comparators (workloads.h:264-298) ----------------

def tensors_close(a: np.ndarray, b: np.ndarray, rel_tol: float = 1e-5) -> bool:
    if a.shape != b.shape:
        return False
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    denom = np.maximum(np.maximum(np.abs(a64), np.abs(b64)), 1.0)
    return bool(np.all(np.abs(a64 - b64) <= rel_tol * denom))


def tensors_close_dot(a: np.ndarray, b: np.ndarray, abs_sum: np.ndarray, rel_tol: float = 1e-4,
                      dot_tol: float = 1e-6) -> bool:
    """D2 criterion for reductions evaluated in a different order: each element
    must satisfy tensors_close (|x-y| <= rel_tol*max(|x|,|y|,1)) OR be within
    dot_tol of its dot product's absolute sum sum|a_k*b_k| (`abs_sum`, the
    oracle run on |A|, |B|). A reassociated fp32 sum of K terms is accurate
    relative to sum|a*b|, not to the (possibly cancelled) result; 1e-6 is
    ~16 ulp of fp32."""
    if a.shape != b.shape:
        return False
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    err = np.abs(a64 - b64)
    denom = np.maximum(np.maximum(np.abs(a64), np.abs(b64)), 1.0)
    ok = (err <= rel_tol * denom) | (err <= dot_tol * abs_sum.astype(np.float64))
    return bool(np.all(ok))


def d2_stats(a: np.ndarray, b: np.ndarray, abs_sum: np.ndarray, rel_tol: float = 1e-4,
             dot_tol: float = 1e-6) -> dict:
    """tensors_close_dot, itemised: how many elements pass the plain
    tensors_close bar (rel_tol), how many pass ONLY through the dot-product
    clause, how many fail, and the worst errors of each kind."""
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    err = np.abs(a64 - b64)
    denom = np.maximum(np.maximum(np.abs(a64), np.abs(b64)), 1.0)
    rel_ok = err <= rel_tol * denom
    dot_ok = err <= dot_tol * abs_sum.astype(np.float64)
    return {"elements": int(a.size), "bitwise_equal": int(np.sum(a64 == b64)),
            "rel_ok": int(np.sum(rel_ok)), "dot_clause_only": int(np.sum(dot_ok & ~rel_ok)),
            "failed": int(np.sum(~(rel_ok | dot_ok))),
            "max_rel_err": float(np.max(err / denom)) if a.size else 0.0,
            "max_err_over_abs_sum": float(np.max(err / np.maximum(abs_sum, 1e-30))) if a.size else 0.0}


def tensors_bitwise_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """Value equality as the reference defines it (get_f compared with !=, so
    +0 == -0)."""
    return a.shape == b.shape and bool(np.all(a.astype(np.float64) == b.astype(np.float64)))


# ---------------- the C restatement ----------------

_lib_oracle = None
_lib_ref = None


def _oracle():
    global _lib_oracle
    if _lib_oracle is None:
        lib = ctypes.CDLL(ORACLE_LIB)
        f32p = ctypes.POINTER(ctypes.c_float)
        lib.tir_oracle_gmm.argtypes = [f32p, f32p, f32p, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        lib.tir_oracle_conv.argtypes = [ctypes.POINTER(ConvDesc), f32p, f32p, f32p, ctypes.c_int,
                                        ctypes.c_int]
        _lib_oracle = lib
    return _lib_oracle


def _fp(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def gmm(A: np.ndarray, B: np.ndarray, C: np.ndarray | None = None, threads: int = 1) -> np.ndarray:
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    M, K = A.shape
    N = B.shape[1]
    out = np.zeros((M, N), np.float32) if C is None else np.array(C, np.float32, copy=True)
    rc = _oracle().tir_oracle_gmm(_fp(A), _fp(B), _fp(out), M, N, K, int(C is not None), threads)
    assert rc == 0
    return out


def conv(spec: ConvSpec, X: np.ndarray, W: np.ndarray, Y: np.ndarray | None = None,
         threads: int = 1) -> np.ndarray:
    X = np.ascontiguousarray(X, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    out = np.zeros(spec.y_shape(), np.float32) if Y is None else np.array(Y, np.float32, copy=True)
    d = ConvDesc.from_spec(spec)
    rc = _oracle().tir_oracle_conv(ctypes.byref(d), _fp(X), _fp(W), _fp(out), int(Y is not None),
                                   threads)
    if rc != 0:
        raise ValueError(f"oracle rejected {spec}")
    return out


def epilogue(Y: np.ndarray, bias: np.ndarray | None = None, relu: bool = False) -> np.ndarray:
    """Fused-epilogue stage in f32: Y + bias[last dim], then max(v, 0.0) as the
    interpreter evaluates max (std::max, interp.cc:499; the relu block of
    gemm_relu_source, tests/testing/workloads.h:83-88). NaN / -0.0 pass through
    like std::max(v, 0.0) = (v < 0) ? 0 : v."""
    out = np.array(Y, np.float32, copy=True)
    if bias is not None:
        out = (out + np.asarray(bias, np.float32)).astype(np.float32)
    if relu:
        out = np.where(out < 0, np.float32(0), out).astype(np.float32)
    return out


# ---------------- the reference interpreter (oracle/_ref) ----------------

def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def _ref():
    global _lib_ref
    if _lib_ref is None:
        lib = ctypes.CDLL(REF_LIB)
        f32p = ctypes.POINTER(ctypes.c_float)
        lib.tirref_run.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(f32p), f32p,
                                   ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_int64)]
        lib.tirref_run_many.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int,
                                        ctypes.POINTER(f32p), ctypes.POINTER(f32p),
                                        ctypes.POINTER(ctypes.c_int64),
                                        ctypes.POINTER(ctypes.c_double)]
        lib.tirref_last_error.restype = ctypes.c_char_p
        _lib_ref = lib
    return _lib_ref


def ref_run(ir_text: str, inputs, out_shape) -> tuple[np.ndarray, float]:
    """tir::run(parse_text(ir_text), inputs) -> (first output, wall seconds)."""
    lib = _ref()
    ins = [np.ascontiguousarray(x, np.float32) for x in inputs]
    arr = (ctypes.POINTER(ctypes.c_float) * len(ins))(*[_fp(x) for x in ins])
    out = np.zeros(out_shape, np.float32)
    wall = ctypes.c_double(0)
    calls = ctypes.c_int64(0)
    rc = lib.tirref_run(ir_text.encode(), len(ins), arr, _fp(out), out.size, ctypes.byref(wall),
                        ctypes.byref(calls))
    if rc != 0:
        raise RuntimeError(lib.tirref_last_error().decode())
    return out, wall.value


def ref_run_many(ir_texts, inputs) -> float:
    """Runs independent programs concurrently (one thread each) on shared
    inputs; returns wall seconds. Used for the sharded CPU baseline."""
    lib = _ref()
    ins = [np.ascontiguousarray(x, np.float32) for x in inputs]
    n = len(ir_texts)
    ptrs = [_fp(x) for x in ins] * n
    arr = (ctypes.POINTER(ctypes.c_float) * len(ptrs))(*ptrs)
    texts = (ctypes.c_char_p * n)(*[t.encode() for t in ir_texts])
    wall = ctypes.c_double(0)
    rc = lib.tirref_run_many(n, texts, len(ins), arr, None, None, ctypes.byref(wall))
    if rc != 0:
        raise RuntimeError(lib.tirref_last_error().decode())
    return wall.value


def timed(fn, *a, **kw):
    t0 = time.perf_counter()
    r = fn(*a, **kw)
    return r, time.perf_counter() - t0
