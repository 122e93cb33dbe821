"""Python host mirror of the B200 intrinsic library (ctypes over include/tir_b200.h).

The reference's interface for this path is the intrinsic host-kernel registry:
a tensorized block calls a named intrinsic, the interpreter hands the kernel the
views [writes[0], reads...] and the kernel accumulates into the output window
(/root/reference/proj/include/tir/interp.h:120-139, src/interp.cc:360-383).
This module exposes the same operators to Python callers on device tensors
(torch is used only for device memory and streams) and on host numpy buffers,
and raises TirError with the reference's error kinds (include/tir/ir.h:33-48).

There is no CPU fallback: if libtir_b200.so is missing or no GPU is visible,
every compute call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, replace

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# TIR_B200_LIB overrides the library path (A/B timing of two builds of the same ABI)
LIB_PATH = os.environ.get("TIR_B200_LIB") or os.path.join(PKG, "lib", "libtir_b200.so")

OK, ERR_VALUE, ERR_UNSUPPORTED, ERR_CUDA = 0, 1, 2, 3
_KINDS = {ERR_VALUE: "ValueError", ERR_UNSUPPORTED: "UnsupportedShape", ERR_CUDA: "CudaError"}
OP_CODES = {"GMM": 0, "C1D": 1, "C2D": 2, "C3D": 3, "DIL": 4, "GRP": 5, "T2D": 6, "DEP": 7}


class TirError(RuntimeError):
    """Mirror of tir::Error(kind, msg) (ir.h:33-48)."""

    def __init__(self, kind: str, message: str):
        super().__init__(f"{kind}: {message}")
        self.kind = kind
        self.message = message


class ConvDesc(ctypes.Structure):
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


@dataclass(frozen=True)
class Conv:
    """Convolution geometry (tir_b200_conv_desc). Spatial tuples are (D, H, W)."""

    op: str = "C2D"
    n: int = 1
    in_dhw: tuple = (1, 1, 1)
    ci: int = 1
    co: int = 1
    k: tuple = (1, 1, 1)
    s: tuple = (1, 1, 1)
    p: tuple = (0, 0, 0)
    d: tuple = (1, 1, 1)
    groups: int = 1
    transposed: bool = False

    def desc(self) -> ConvDesc:
        return ConvDesc(OP_CODES[self.op], int(self.transposed), self.n, *self.in_dhw, self.ci,
                        self.co, *self.k, *self.s, *self.p, *self.d, self.groups)

    @property
    def spatial_rank(self) -> int:
        return 1 if self.op == "C1D" else 3 if self.op == "C3D" else 2

    def out_dhw(self) -> tuple:
        out = (ctypes.c_int64 * 3)()
        d = self.desc()
        _check(lib().tir_b200_conv_out_shape(ctypes.byref(d), out))
        return tuple(out)

    def x_shape(self):
        r = self.spatial_rank
        return (self.n, *self.in_dhw[3 - r:], self.ci)

    def w_shape(self):
        r = self.spatial_rank
        if self.op == "DEP":
            return (*self.k[3 - r:], self.co)
        return (*self.k[3 - r:], self.ci // self.groups, self.co)

    def y_shape(self):
        r = self.spatial_rank
        return (self.n, *self.out_dhw()[3 - r:], self.co)

    def with_(self, **kw) -> "Conv":
        return replace(self, **kw)


class BatchDesc(ctypes.Structure):
    """tir_b200_batch_desc: per-problem coordinates base + z1*step1 + z2*step2."""
    _fields_ = [("z1n", ctypes.c_int64), ("z2n", ctypes.c_int64)] + [
        (f"{t}_{d}", ctypes.c_int64 * 3) for t in "abc" for d in ("row", "col")] + [("b_kmajor", ctypes.c_int64)]


class Epilogue(ctypes.Structure):
    """tir_b200_epilogue: optional per-column fp32 bias, fp16 residual, then an
    activation (include/tir_b200.h)."""
    _fields_ = [("bias", ctypes.c_void_p), ("relu", ctypes.c_int32), ("residual", ctypes.c_void_p)]


ACT_NONE, ACT_RELU, ACT_RELU6, ACT_GELU = 0, 1, 2, 3
_ACTS = {None: 0, False: 0, True: 1, "none": 0, "relu": 1, "relu6": 2, "gelu": 3, 0: 0, 1: 1, 2: 2, 3: 3}


_lib = None


def lib() -> ctypes.CDLL:
    """Loads libtir_b200.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TirError("CudaError", f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.tir_b200_last_error.restype = ctypes.c_char_p
        L.tir_b200_launch_count.restype = i64
        L.tir_b200_conv_out_shape.argtypes = [ctypes.POINTER(ConvDesc), ctypes.POINTER(i64)]
        L.tir_b200_gmm.argtypes = [vp, vp, vp, vp, i64, i64, i64, i32, i32, vp]
        L.tir_b200_conv.argtypes = [ctypes.POINTER(ConvDesc), vp, vp, vp, vp, i32, i32, vp]
        ep = ctypes.POINTER(Epilogue)
        L.tir_b200_gmm_ex.argtypes = [vp, vp, vp, vp, i64, i64, i64, i32, i32, ep, vp]
        L.tir_b200_conv_ex.argtypes = [ctypes.POINTER(ConvDesc), vp, vp, vp, vp, i32, i32, ep, vp]
        L.tir_b200_gmm_host.argtypes = [vp, vp, vp, i64, i64, i64, i32]
        L.tir_b200_conv_host.argtypes = [ctypes.POINTER(ConvDesc), vp, vp, vp, i32]
        L.tir_b200_gmm_host_f32.argtypes = [vp, vp, vp, i64, i64, i64, i32]
        L.tir_b200_maxpool2d.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, vp]
        L.tir_b200_avgpool_global.argtypes = [vp, vp, i64, i64, i64, vp]
        L.tir_b200_layernorm.argtypes = [vp, vp, vp, vp, i64, i64, ctypes.c_float, vp]
        L.tir_b200_softmax.argtypes = [vp, vp, i64, i64, ctypes.c_float, vp]
        L.tir_b200_gmm_batched.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, i64, i64, i64, i64,
                                           ctypes.POINTER(BatchDesc), i32, ctypes.POINTER(Epilogue), vp]
        L.tir_b200_conv_host_f32.argtypes = [ctypes.POINTER(ConvDesc), vp, vp, vp, i32]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != OK:
        raise TirError(_KINDS.get(rc, "InternalError"), lib().tir_b200_last_error().decode())


def launch_count() -> int:
    return int(lib().tir_b200_launch_count())


def reset_launch_count() -> None:
    lib().tir_b200_reset_launch_count()


def set_option(name: str, value: int) -> None:
    """Planner switch (csrc/options.h): tile shape / pipeline / epilogue flavour, never results."""
    _check(lib().tir_b200_set_option(name.encode(), int(value)))


def get_option(name: str) -> int:
    v = ctypes.c_int(0)
    _check(lib().tir_b200_get_option(name.encode(), ctypes.byref(v)))
    return v.value


# ---------------------------------------------------------------- device tensors

def _torch():
    import torch  # plumbing only: device memory + streams

    return torch


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need(t, dtype, shape, name):
    torch = _torch()
    if not t.is_cuda:
        raise TirError("ValueError", f"{name} must be a CUDA tensor")
    if t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise TirError("ValueError", f"{name}: expected contiguous {dtype} {tuple(shape)}, got "
                                     f"{t.dtype} {tuple(t.shape)}")
    del torch


def _epilogue(bias, relu, cols, device, residual=None, out_shape=None):
    """Builds the C-ABI epilogue; None when nothing is requested. `relu` is a bool
    (ReLU) or an activation name/code: "relu", "relu6", "gelu"."""
    if relu not in _ACTS:
        raise TirError("ValueError", f"unknown activation {relu!r}")
    act = _ACTS[relu]
    if bias is None and not act and residual is None:
        return None
    torch = _torch()
    if bias is not None:
        _need(bias, torch.float32, (cols,), "bias")
        if bias.device != device:
            raise TirError("ValueError", "bias must live on the operands' device")
    if residual is not None:
        _need(residual, torch.float16, out_shape, "residual")
        if residual.device != device:
            raise TirError("ValueError", "residual must live on the operands' device")
    return Epilogue(bias.data_ptr() if bias is not None else None, act,
                    residual.data_ptr() if residual is not None else None)


def gmm(A, B, C=None, *, accumulate: bool = False, out_f16: bool = False, bias=None,
        relu=False, residual=None, stream=None):
    """C (+)= A @ B with A [M,K] fp16, B [K,N] fp16 (N contiguous), fp32 accumulation.
    Optional fused epilogue: C = act((C +) A @ B + bias[N] + residual[M,N]), act from
    `relu` (True / "relu", "relu6", "gelu"). Returns C ([M,N] fp32, or fp16 if out_f16)."""
    torch = _torch()
    M, K = A.shape
    N = B.shape[1]
    _need(A, torch.float16, (M, K), "A")
    _need(B, torch.float16, (K, N), "B")
    if C is None:
        if accumulate:
            raise TirError("ValueError", "accumulate needs C")
        C = torch.empty((M, N), dtype=torch.float16 if out_f16 else torch.float32, device=A.device)
    _need(C, torch.float16 if out_f16 else torch.float32, (M, N), "C")
    if accumulate and out_f16:
        raise TirError("ValueError", "accumulate requires an fp32 C")
    epi = _epilogue(bias, relu, N, A.device, residual, (M, N))
    if epi is None:
        _check(lib().tir_b200_gmm(_ptr(A), _ptr(B), _ptr(C) if accumulate else None, _ptr(C), M, N, K,
                                  int(accumulate), int(out_f16), _stream(stream)))
    else:
        _check(lib().tir_b200_gmm_ex(_ptr(A), _ptr(B), _ptr(C) if accumulate else None, _ptr(C), M, N,
                                     K, int(accumulate), int(out_f16), ctypes.byref(epi),
                                     _stream(stream)))
    return C


def conv(spec: Conv, X, W, Y=None, *, accumulate: bool = False, out_f16: bool = False,
         bias=None, relu=False, residual=None, stream=None):
    """Y (+)= conv(X, W) for C1D/C2D/C3D/DIL/GRP/T2D/DEP (layouts: include/tir_b200.h).
    Optional fused epilogue: Y = act((Y +) conv(X, W) + bias[CO] + residual), residual
    fp16 with Y's shape (not for DEP); act from `relu` (True / "relu", "relu6", "gelu")."""
    torch = _torch()
    _need(X, torch.float16, spec.x_shape(), "X")
    _need(W, torch.float16, spec.w_shape(), "W")
    ydt = torch.float16 if out_f16 else torch.float32
    if Y is None:
        if accumulate:
            raise TirError("ValueError", "accumulate needs Y")
        Y = torch.empty(spec.y_shape(), dtype=ydt, device=X.device)
    _need(Y, ydt, spec.y_shape(), "Y")
    if accumulate and out_f16:
        raise TirError("ValueError", "accumulate requires an fp32 Y")
    d = spec.desc()
    epi = _epilogue(bias, relu, spec.co, X.device, residual, spec.y_shape())
    if epi is None:
        _check(lib().tir_b200_conv(ctypes.byref(d), _ptr(X), _ptr(W), _ptr(Y) if accumulate else None,
                                   _ptr(Y), int(accumulate), int(out_f16), _stream(stream)))
    else:
        _check(lib().tir_b200_conv_ex(ctypes.byref(d), _ptr(X), _ptr(W),
                                      _ptr(Y) if accumulate else None, _ptr(Y), int(accumulate),
                                      int(out_f16), ctypes.byref(epi), _stream(stream)))
    return Y


# ---------------------------------------------------------------- network glue

def maxpool2d(X, k: int, s: int, p: int, Y=None, *, stream=None):
    """NHWC fp16 max pooling (padding never wins); returns Y [N, OH, OW, C]."""
    torch = _torch()
    n, h, w, c = X.shape
    _need(X, torch.float16, (n, h, w, c), "X")
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    if Y is None:
        Y = torch.empty((n, oh, ow, c), dtype=torch.float16, device=X.device)
    _need(Y, torch.float16, (n, oh, ow, c), "Y")
    _check(lib().tir_b200_maxpool2d(_ptr(X), _ptr(Y), n, h, w, c, k, s, p, _stream(stream)))
    return Y


def avgpool_global(X, Y=None, *, stream=None):
    """NHWC fp16 [N, H, W, C] -> [N, C] fp16 mean over pixels (fp32 sum)."""
    torch = _torch()
    n, h, w, c = X.shape
    _need(X, torch.float16, (n, h, w, c), "X")
    if Y is None:
        Y = torch.empty((n, c), dtype=torch.float16, device=X.device)
    _need(Y, torch.float16, (n, c), "Y")
    _check(lib().tir_b200_avgpool_global(_ptr(X), _ptr(Y), n, h * w, c, _stream(stream)))
    return Y


def layernorm(X, gamma, beta, eps: float = 1e-12, Y=None, *, stream=None):
    """Row LayerNorm of fp16 X [rows, cols] with fp32 gamma/beta; fp16 out."""
    torch = _torch()
    rows, cols = X.shape
    _need(X, torch.float16, (rows, cols), "X")
    _need(gamma, torch.float32, (cols,), "gamma")
    _need(beta, torch.float32, (cols,), "beta")
    if Y is None:
        Y = torch.empty_like(X)
    _need(Y, torch.float16, (rows, cols), "Y")
    _check(lib().tir_b200_layernorm(_ptr(X), _ptr(Y), _ptr(gamma), _ptr(beta), rows, cols, eps,
                                    _stream(stream)))
    return Y


def softmax(X, scale: float = 1.0, Y=None, *, stream=None):
    """Row softmax(scale * X) of fp16 X [rows, cols]; fp16 out."""
    torch = _torch()
    rows, cols = X.shape
    _need(X, torch.float16, (rows, cols), "X")
    if Y is None:
        Y = torch.empty_like(X)
    _need(Y, torch.float16, (rows, cols), "Y")
    _check(lib().tir_b200_softmax(_ptr(X), _ptr(Y), rows, cols, scale, _stream(stream)))
    return Y


def gmm_batched(A, B, C, M: int, N: int, K: int, z: tuple, a: tuple, b: tuple, c: tuple, *,
                b_kmajor: bool = False, out_f16: bool = True, bias=None, relu=False, residual=None,
                stream=None):
    """Batched GMM over strided windows of 2-D tensors (include/tir_b200.h):
    problem (z1, z2) computes C[cr + m, cc + n] = sum_k A[ar + m, ac + k] * B[br + k, bc + n]
    (b_kmajor: B[br + n, bc + k]), each coordinate given as ((base, step1, step2) for rows,
    (base, step1, step2) for cols)."""
    torch = _torch()
    _need(A, torch.float16, A.shape, "A")
    _need(B, torch.float16, B.shape, "B")
    _need(C, torch.float16 if out_f16 else torch.float32, C.shape, "C")
    d = BatchDesc()
    d.z1n, d.z2n = z
    for name, (rows, cols) in zip("abc", (a, b, c)):
        getattr(d, f"{name}_row")[:] = rows
        getattr(d, f"{name}_col")[:] = cols
    d.b_kmajor = int(bool(b_kmajor))
    epi = _epilogue(bias, relu, N, A.device, residual, tuple(C.shape))
    _check(lib().tir_b200_gmm_batched(_ptr(A), A.shape[0], A.shape[1], _ptr(B), B.shape[0], B.shape[1],
                                      _ptr(C), C.shape[0], C.shape[1], M, N, K, ctypes.byref(d),
                                      int(out_f16), ctypes.byref(epi) if epi is not None else None,
                                      _stream(stream)))
    return C


# ---------------------------------------------------------------- host buffers

def _np_ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def gmm_host(A: np.ndarray, B: np.ndarray, C: np.ndarray | None = None,
             accumulate: bool = False) -> np.ndarray:
    """Host fp16 (or f32 holding fp16 values, as the interpreter stores F16)
    inputs -> host fp32 C. Synchronous: H2D, kernel, D2H."""
    M, K = A.shape
    N = B.shape[1]
    if C is None:
        C = np.zeros((M, N), np.float32)
    assert C.dtype == np.float32 and C.flags.c_contiguous
    if A.dtype == np.float16 and B.dtype == np.float16:
        A, B = np.ascontiguousarray(A), np.ascontiguousarray(B)
        _check(lib().tir_b200_gmm_host(_np_ptr(A), _np_ptr(B), _np_ptr(C), M, N, K, int(accumulate)))
    else:
        A = np.ascontiguousarray(A, np.float32)
        B = np.ascontiguousarray(B, np.float32)
        _check(lib().tir_b200_gmm_host_f32(_np_ptr(A), _np_ptr(B), _np_ptr(C), M, N, K,
                                           int(accumulate)))
    return C


def conv_host(spec: Conv, X: np.ndarray, W: np.ndarray, Y: np.ndarray | None = None,
              accumulate: bool = False) -> np.ndarray:
    if Y is None:
        Y = np.zeros(spec.y_shape(), np.float32)
    assert Y.dtype == np.float32 and Y.flags.c_contiguous
    d = spec.desc()
    if X.dtype == np.float16 and W.dtype == np.float16:
        X, W = np.ascontiguousarray(X), np.ascontiguousarray(W)
        _check(lib().tir_b200_conv_host(ctypes.byref(d), _np_ptr(X), _np_ptr(W), _np_ptr(Y),
                                        int(accumulate)))
    else:
        X = np.ascontiguousarray(X, np.float32)
        W = np.ascontiguousarray(W, np.float32)
        _check(lib().tir_b200_conv_host_f32(ctypes.byref(d), _np_ptr(X), _np_ptr(W), _np_ptr(Y),
                                            int(accumulate)))
    return Y


# ---------------------------------------------------------------- the paper's shapes

PAPER_SHAPES = {
    "C1D": Conv("C1D", n=16, in_dhw=(1, 1, 256), ci=64, co=128, k=(1, 1, 3), s=(1, 1, 2), p=(0, 0, 1)),
    "C2D": Conv("C2D", n=16, in_dhw=(1, 56, 56), ci=64, co=64, k=(1, 3, 3), s=(1, 1, 1), p=(0, 1, 1)),
    "C3D": Conv("C3D", n=16, in_dhw=(16, 224, 224), ci=3, co=64, k=(7, 7, 7), s=(2, 2, 2), p=(3, 3, 3)),
    "DIL": Conv("DIL", n=16, in_dhw=(1, 224, 224), ci=3, co=64, k=(1, 7, 7), s=(1, 2, 2), p=(0, 3, 3),
                d=(1, 2, 2)),
    "GRP": Conv("GRP", n=16, in_dhw=(1, 56, 56), ci=64, co=128, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1),
                groups=4),
    "T2D": Conv("T2D", n=16, in_dhw=(1, 4, 4), ci=512, co=256, k=(1, 4, 4), s=(1, 2, 2), p=(0, 1, 1),
                transposed=True),
    "DEP": Conv("DEP", n=16, in_dhw=(1, 112, 112), ci=32, co=32, k=(1, 3, 3), s=(1, 1, 1), p=(0, 1, 1),
                groups=32),
}
GMM_SHAPE = (1024, 1024, 1024)


def useful_macs(spec: Conv) -> int:
    """MACs of the unpadded math (T2D: useful, structural zeros excluded)."""
    kd, kh, kw = spec.k
    if spec.transposed:
        return spec.n * int(np.prod(spec.in_dhw)) * spec.ci * spec.co * kd * kh * kw // spec.groups
    od, oh, ow = spec.out_dhw()
    return spec.n * od * oh * ow * spec.co * kd * kh * kw * (spec.ci // spec.groups)


def compulsory_bytes(spec: Conv, out_bytes: int = 4) -> int:
    """Each input once + weights once + output once at actual dtypes."""
    x = int(np.prod(spec.x_shape())) * 2
    w = int(np.prod(spec.w_shape())) * 2
    y = int(np.prod(spec.y_shape())) * out_bytes
    return x + w + y
