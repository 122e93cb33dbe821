"""Build recipe for the native libraries (run by __graft_entry__.build()).

  lib/libtir_b200.so          the product: sm_100a kernels + the C-ABI of include/tir_b200.h
  lib/libtir_b200_adapter.so  the reference-side HostKernel adapter (adapter/), compiled
                              against the unmodified reference headers and linked with
                              the reference interpreter built in oracle/_ref — only when
                              /root/reference is present (this container); tests load it.

Everything is built in-tree so the .so files travel to the GPU box with the
repo snapshot. nvcc flags: -gencode arch=compute_100a,code=sm_100a (plain
-arch=sm_100a also emits a compute_100 PTX pass that rejects tcgen05).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
REF = "/root/reference/proj"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
    "-Xcompiler", "-Wall",
]

SOURCES = ["csrc/tir_b200.cu"]
HEADERS = ["csrc/ptx.cuh", "csrc/igemm.cuh", "csrc/halo.cuh", "csrc/dep.cuh", "csrc/prep.cuh", "csrc/netops.cuh",
           "csrc/rowpack.cuh", "csrc/options.h",
           "../include/tir_b200.h"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd):
    print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)


def build_core(force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    out = os.path.join(LIB, "libtir_b200.so")
    deps = [os.path.join(PKG, s) for s in SOURCES + HEADERS]
    if force or _stale(out, deps):
        _run([NVCC, *NVCC_FLAGS, "-o", out, *[os.path.join(PKG, s) for s in SOURCES],
              "-lcudart"])
    return out


def build_adapter(force: bool = False) -> str | None:
    """The HostKernel adapter needs the reference's headers and interpreter
    (oracle/_ref/libtirkit.so); skipped where /root/reference is absent."""
    ref_lib = os.path.join(ROOT, "oracle", "_ref", "libtirkit.so")
    out = os.path.join(LIB, "libtir_b200_adapter.so")
    adir = os.path.join(PKG, "adapter")
    srcs = [os.path.join(adir, f) for f in ("tir_b200_adapter.cc", "tir_b200_tensorize.cc")]
    hdrs = [os.path.join(adir, f) for f in ("tir_b200_adapter.h", "tir_b200_tensorize.h")]
    if not (os.path.isdir(REF) and os.path.exists(ref_lib) and all(map(os.path.exists, srcs))):
        return out if os.path.exists(out) else None
    if force or _stale(out, srcs + hdrs + [os.path.join(LIB, "libtir_b200.so"), ref_lib]):
        _run(["g++", "-std=gnu++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra",
              f"-I{REF}/include", f"-I{ROOT}/include", f"-I{ROOT}/oracle/_ref/vendor",
              "-o", out, *srcs,
              f"-L{LIB}", "-ltir_b200", f"-L{ROOT}/oracle/_ref", "-ltirkit",
              "-Wl,-rpath,$ORIGIN", "-Wl,-rpath,$ORIGIN/../../oracle/_ref"])
    return out


def build_oracle() -> None:
    """oracle/Makefile: the C restatement always; the reference interpreter
    (oracle/_ref) when /root/reference is present."""
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8", "all"])


def build_all(force: bool = False) -> None:
    build_oracle()
    build_core(force)
    build_adapter(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
