"""IR-text generators for the paper's operator set — TEST INFRASTRUCTURE.

Emits programs in the reference grammar (parse_text, /root/reference/proj/src/parser.cc:801)
that the reference interpreter (tir::run, src/interp.cc:579) executes as the
oracle. The shapes of the three ops the reference ships sources for follow
them exactly (tests/testing/workloads.h): GMM = matmul_source (:35-58),
C2D = conv2d_source (:95-130, NHWC x HWIO), DEP = depthwise_source (:133-166,
weights [KH,KW,C]). The build generalises them:
  * fp16 operands with explicit f32(...) casts — make_binary rejects mixed
    dtypes (src/ir.cc:88-91); F16 is an f32 tag (ir.cc:36-47);
  * batch N, stride, dilation and zero padding via
    select(in-bounds, f32(A[..]), 0.0) — only the taken branch is evaluated
    (src/interp.cc:463-466);
  * groups (GRP: channel (vco / (CO/G)) * (CI/G) + vrc), 1-D (NLC) and 3-D (NDHWC);
  * T2D in gather form: select((o + p - k d) % s == 0 and in bounds, A[(o+p-k d)/s], 0).
Reduction loop order is the reference's: (rd,) rh, rw, rc innermost.

`rows=(r0, r1)` restricts the outermost output loop (GMM: M rows; conv: the
flattened (n, od, oh) rows) to a slice. Every output element keeps its own
reduction order, so slices are bit-identical to the full program; the CPU
baseline shards work this way.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class ConvSpec:
    """Mirror of tir_b200_conv_desc (include/tir_b200.h)."""

    op: str = "C2D"          # GMM C1D C2D C3D DIL GRP T2D DEP
    n: int = 1
    in_dhw: tuple = (1, 8, 8)
    ci: int = 4
    co: int = 8
    k: tuple = (1, 3, 3)
    s: tuple = (1, 1, 1)
    p: tuple = (0, 0, 0)
    d: tuple = (1, 1, 1)
    groups: int = 1
    transposed: bool = False

    @property
    def spatial_rank(self) -> int:
        if self.op == "C1D":
            return 1
        if self.op == "C3D":
            return 3
        return 2

    def out_dhw(self) -> tuple:
        out = []
        for i, k, s, p, d in zip(self.in_dhw, self.k, self.s, self.p, self.d):
            if self.transposed:
                o = (i - 1) * s - 2 * p + d * (k - 1) + 1
            else:
                o = (i + 2 * p - d * (k - 1) - 1) // s + 1
            if o < 1:
                raise ValueError(f"empty output for {self}")
            out.append(o)
        return tuple(out)

    @property
    def cig(self) -> int:
        return self.ci // self.groups

    @property
    def cog(self) -> int:
        return self.co // self.groups

    def x_shape(self) -> tuple:
        r = self.spatial_rank
        return (self.n, *self.in_dhw[3 - r:], self.ci)

    def w_shape(self) -> tuple:
        r = self.spatial_rank
        if self.op == "DEP":
            return (*self.k[3 - r:], self.co)
        return (*self.k[3 - r:], self.cig, self.co)

    def y_shape(self) -> tuple:
        r = self.spatial_rank
        return (self.n, *self.out_dhw()[3 - r:], self.co)

    def macs(self) -> int:
        """Useful MACs (padding / structural zeros excluded for T2D)."""
        od, oh, ow = self.out_dhw()
        kd, kh, kw = self.k
        if self.transposed:
            dd, dh, dw = self.in_dhw
            return self.n * dd * dh * dw * self.ci * self.co * kd * kh * kw // self.groups
        return self.n * od * oh * ow * self.co * kd * kh * kw * self.cig

    def flops(self) -> int:
        return 2 * self.macs()


def _dims(names, shape):
    return ", ".join(f"{d}" for d in shape)


def gmm_source(m: int, n: int, k: int, rows=None, name: str = "gmm") -> str:
    """f16 x f16 -> f32 matmul, matmul_source (workloads.h:35-58) with casts."""
    r0, r1 = rows if rows else (0, m)
    bind = f"i + {r0}" if r0 else "i"
    return (
        f"func {name}(A: f16[{m}, {k}], B: f16[{k}, {n}], C: f32[{m}, {n}]) {{\n"
        f"  block root() {{\n"
        f"    for i in 0..{r1 - r0} {{\n"
        f"      for j in 0..{n} {{\n"
        f"        for k in 0..{k} {{\n"
        f"          block gemm(spatial vi: {m} = {bind}, spatial vj: {n} = j, reduce vk: {k} = k) "
        f"reads(A[vi +: 1, vk +: 1], B[vk +: 1, vj +: 1]) writes(C[vi +: 1, vj +: 1]) {{\n"
        f"            init {{\n"
        f"              C[vi, vj] = 0.0\n"
        f"            }}\n"
        f"            C[vi, vj] = C[vi, vj] + f32(A[vi, vk])*f32(B[vk, vj])\n"
        f"          }}\n"
        f"        }}\n"
        f"      }}\n"
        f"    }}\n"
        f"  }}\n"
        f"}}\n"
    )


def conv_source(spec: ConvSpec, rows=None, name: str | None = None, cols=None) -> str:
    """Scalar program for C1D/C2D/C3D/DIL/GRP/T2D/DEP (see module doc). `cols`
    restricts the innermost output spatial loop (ow) to [c0, c1)."""
    r = spec.spatial_rank
    name = name or spec.op.lower()
    od, oh, ow = spec.out_dhw()
    out_sp = (od, oh, ow)[3 - r:]
    in_sp = spec.in_dhw[3 - r:]
    ks = spec.k[3 - r:]
    ss = spec.s[3 - r:]
    ps = spec.p[3 - r:]
    ds = spec.d[3 - r:]
    sp_names = ["d", "h", "w"][3 - r:]
    x_shape, w_shape, y_shape = spec.x_shape(), spec.w_shape(), spec.y_shape()
    dep = spec.op == "DEP"
    if dep and (spec.groups != spec.ci or spec.ci != spec.co):
        raise ValueError("DEP requires groups == ci == co")

    # Loop nest: n, spatial outputs, co, then reductions (r<sp>), rc.
    # The outermost output rows (n, od?, oh?) are flattened for slicing.
    row_dims = [("n", spec.n)] + list(zip(sp_names[:-1], out_sp[:-1]))
    total_rows = 1
    for _, e in row_dims:
        total_rows *= e
    r0, r1 = rows if rows else (0, total_rows)

    lines = []
    ind = "    "
    lines.append(f"for row in 0..{r1 - r0} {{")
    depth = 1
    c0, c1 = cols if cols else (0, out_sp[-1])
    lines.append(ind * depth + f"for {sp_names[-1]} in 0..{c1 - c0} {{")
    depth += 1
    lines.append(ind * depth + f"for co in 0..{spec.co} {{")
    depth += 1
    for nm, kk in zip(sp_names, ks):
        lines.append(ind * depth + f"for r{nm} in 0..{kk} {{")
        depth += 1
    if not dep:
        lines.append(ind * depth + f"for rc in 0..{spec.cig} {{")
        depth += 1

    # Bindings: decompose the flattened row index.
    row_expr = f"(row + {r0})" if r0 else "row"
    binds = []
    stride = 1
    decomp = {}
    for nm, e in reversed(row_dims):
        if stride == 1:
            decomp[nm] = f"{row_expr} % {e}" if nm != "n" else f"{row_expr}"
        else:
            decomp[nm] = f"{row_expr} / {stride} % {e}" if nm != "n" else f"{row_expr} / {stride}"
        stride *= e
    if len(row_dims) == 1:
        decomp["n"] = row_expr
    binds.append(f"spatial vn: {spec.n} = {decomp['n']}")
    for nm, e in zip(sp_names[:-1], out_sp[:-1]):
        binds.append(f"spatial v{nm}: {e} = {decomp[nm]}")
    binds.append(f"spatial v{sp_names[-1]}: {out_sp[-1]} = {sp_names[-1]}" + (f" + {c0}" if c0 else ""))
    binds.append(f"spatial vco: {spec.co} = co")
    for nm, kk in zip(sp_names, ks):
        binds.append(f"reduce vr{nm}: {kk} = r{nm}")
    if not dep:
        binds.append(f"reduce vrc: {spec.cig} = rc")

    # Input coordinate expressions + in-bounds condition.
    in_idx, conds = [], []
    for nm, I, k_, s_, p_, d_ in zip(sp_names, in_sp, ks, ss, ps, ds):
        tap = f"vr{nm}" if d_ == 1 else f"vr{nm}*{d_}"
        if spec.transposed:
            t = f"(v{nm} + {p_} - {tap})"
            idx = f"{t} / {s_}" if s_ != 1 else t
            if s_ != 1:
                conds.append(f"{t} % {s_} == 0")
        else:
            base = f"v{nm}" if s_ == 1 else f"v{nm}*{s_}"
            idx = f"{base} + {tap}" + (f" - {p_}" if p_ else "")
        in_idx.append(idx)
        if spec.transposed or p_ > 0:  # without padding every forward tap is in bounds
            conds.append(f"{idx} >= 0")
            conds.append(f"{idx} < {I}")
    if dep:
        chan = "vco"
    elif spec.groups == 1:
        chan = "vrc"
    else:
        chan = f"vco / {spec.cog} * {spec.cig} + vrc"
    a_idx = ", ".join(["vn", *in_idx, chan])
    y_idx = ", ".join(["vn", *[f"v{nm}" for nm in sp_names], "vco"])
    w_idx = ", ".join([*[f"vr{nm}" for nm in sp_names], *([] if dep else ["vrc"]), "vco"])
    a_load = f"f32(A[{a_idx}])"
    if conds:
        a_load = f"select({' and '.join(conds)}, {a_load}, 0.0)"
    a_region = ", ".join(f"0 +: {e}" for e in x_shape)
    w_region = ", ".join(f"{x} +: 1" for x in w_idx.split(", "))
    y_region = ", ".join(f"{x} +: 1" for x in y_idx.split(", "))

    body = (
        f"block conv({', '.join(binds)}) reads(A[{a_region}], B[{w_region}]) "
        f"writes(C[{y_region}]) {{\n"
        f"  init {{\n"
        f"    C[{y_idx}] = 0.0\n"
        f"  }}\n"
        f"  C[{y_idx}] = C[{y_idx}] + {a_load}*f32(B[{w_idx}])\n"
        f"}}"
    )
    for ln in body.split("\n"):
        lines.append(ind * depth + ln)
    while depth > 0:
        depth -= 1
        lines.append(ind * depth + "}")

    header = (
        f"func {name}(A: f16[{_dims(None, x_shape)}], B: f16[{_dims(None, w_shape)}], "
        f"C: f32[{_dims(None, y_shape)}]) {{\n  block root() {{\n"
    )
    return header + "\n".join("    " + ln for ln in lines) + "\n  }\n}\n"


def tensorized_gmm_source(m: int, n: int, k: int, intrin: str = "b200.gmm",
                          tiles=(1, 1, 1), name: str = "gmm_t") -> str:
    """GMM as tensorized blocks calling `intrin` (the CS3 whole-op form, SURVEY
    Appendix; tiled variant mirrors tests/test_interp.cc:162-208). No
    exec_scope annotation: TH-SCOPE would reject a whole-op block
    (validate.cc:432-455)."""
    ti, tj, tk = tiles
    bm, bn, bk = m // ti, n // tj, k // tk
    if bm * ti != m or bn * tj != n or bk * tk != k:
        raise ValueError("tiles must divide the problem")
    return (
        f"func {name}(A: f16[{m}, {k}], B: f16[{k}, {n}], C: f32[{m}, {n}]) {{\n"
        f"  block root() {{\n"
        f"    for io in 0..{ti} {{\n"
        f"      for jo in 0..{tj} {{\n"
        f"        for ko in 0..{tk} {{\n"
        f"          block mm(spatial vio: {ti} = io, spatial vjo: {tj} = jo, reduce vko: {tk} = ko) "
        f"reads(A[vio*{bm} +: {bm}, vko*{bk} +: {bk}], B[vko*{bk} +: {bk}, vjo*{bn} +: {bn}]) "
        f"writes(C[vio*{bm} +: {bm}, vjo*{bn} +: {bn}]) attrs(\"tensorized\" = \"{intrin}\") {{\n"
        f"            {intrin}()\n"
        f"          }}\n"
        f"        }}\n"
        f"      }}\n"
        f"    }}\n"
        f"  }}\n"
        f"}}\n"
    )


def tensorized_conv_source(spec: ConvSpec, intrin: str, name: str = "conv_t") -> str:
    """Whole-op tensorized conv block: views [Y, X, W] in signature order
    (interp.cc:371-373)."""
    x, w, y = spec.x_shape(), spec.w_shape(), spec.y_shape()
    reg = lambda shp: ", ".join(f"0 +: {e}" for e in shp)  # noqa: E731
    return (
        f"func {name}(A: f16[{_dims(None, x)}], B: f16[{_dims(None, w)}], C: f32[{_dims(None, y)}]) {{\n"
        f"  block root() {{\n"
        f"    block op(spatial vo: 1 = 0) reads(A[{reg(x)}], B[{reg(w)}]) writes(C[{reg(y)}]) "
        f"attrs(\"tensorized\" = \"{intrin}\") {{\n"
        f"      {intrin}()\n"
        f"    }}\n"
        f"  }}\n"
        f"}}\n"
    )


def with_epilogue(src: str, out_shape: tuple, bias: bool = False, relu: bool = False) -> str:
    """Adds the fused-epilogue stage to a contraction program:
    the output C becomes an `alloc` intermediate and a second nest writes
    D = max(C + Bias[last dim], 0.0) — the shape of the reference's own
    gemm_relu_source (tests/testing/workloads.h:61-91: alloc C, then
    `D[vi, vj] = max(C[vi, vj], 0.0)`), generalised with an optional f32 bias
    per output column. Inputs become (A, B[, Bias]); the output is D."""
    dims = _dims(None, out_shape)
    head = f"C: f32[{dims}]) {{\n  block root() {{\n"
    if src.count(head) != 1:
        raise ValueError("program does not have the expected C output signature")
    params = (f"Bias: f32[{out_shape[-1]}], " if bias else "") + f"D: f32[{dims}]"
    src = src.replace(head, f"{params}) {{\n  block root() {{\n    alloc C: f32[{dims}]\n")
    tail = "  }\n}\n"
    assert src.endswith(tail)
    body = src[: -len(tail)]
    nd = len(out_shape)
    ind = "  "
    lines = []
    for i, e in enumerate(out_shape):
        lines.append(ind * (2 + i) + f"for e{i} in 0..{e} {{")
    binds = ", ".join(f"spatial u{i}: {e} = e{i}" for i, e in enumerate(out_shape))
    idx = ", ".join(f"u{i}" for i in range(nd))
    reg = ", ".join(f"u{i} +: 1" for i in range(nd))
    reads = f"C[{reg}]" + (f", Bias[u{nd - 1} +: 1]" if bias else "")
    val = f"C[{idx}]" + (f" + Bias[u{nd - 1}]" if bias else "")
    if relu:
        val = f"max({val}, 0.0)"
    d = ind * (2 + nd)
    lines.append(d + f"block epi({binds}) reads({reads}) writes(D[{reg}]) {{")
    lines.append(d + f"  D[{idx}] = {val}")
    lines.append(d + "}")
    for i in reversed(range(nd)):
        lines.append(ind * (2 + i) + "}")
    return body + "\n".join(lines) + "\n" + tail


# ---- the paper's single-op suite (SURVEY §8(d) proposed benchmark shapes) ----

PAPER_SHAPES = {
    "C1D": ConvSpec("C1D", n=16, in_dhw=(1, 1, 256), ci=64, co=128, k=(1, 1, 3), s=(1, 1, 2), p=(0, 0, 1)),
    "C2D": ConvSpec("C2D", n=16, in_dhw=(1, 56, 56), ci=64, co=64, k=(1, 3, 3), s=(1, 1, 1), p=(0, 1, 1)),
    "C3D": ConvSpec("C3D", n=16, in_dhw=(16, 224, 224), ci=3, co=64, k=(7, 7, 7), s=(2, 2, 2), p=(3, 3, 3)),
    "DIL": ConvSpec("DIL", n=16, in_dhw=(1, 224, 224), ci=3, co=64, k=(1, 7, 7), s=(1, 2, 2), p=(0, 3, 3), d=(1, 2, 2)),
    "GRP": ConvSpec("GRP", n=16, in_dhw=(1, 56, 56), ci=64, co=128, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=4),
    "T2D": ConvSpec("T2D", n=16, in_dhw=(1, 4, 4), ci=512, co=256, k=(1, 4, 4), s=(1, 2, 2), p=(0, 1, 1), transposed=True),
    "DEP": ConvSpec("DEP", n=16, in_dhw=(1, 112, 112), ci=32, co=32, k=(1, 3, 3), s=(1, 1, 1), p=(0, 1, 1), groups=32),
}

GMM_SHAPE = (1024, 1024, 1024)


def small(spec: ConvSpec, **kw) -> ConvSpec:
    return replace(spec, **kw)


def conv_source_direct(spec: ConvSpec, name: str | None = None) -> str:
    """Forward, groups = 1 convolution with one loop per block iterator and
    per-element read regions (A[vn +: 1, <input index> +: 1, ..., vrc +: 1]).
    This is the form the reference's Schedule::pad_block accepts (trivial loop
    bindings, directly indexed padded operands; schedule_block.cc:1186-1260),
    used to express the channel pad CI -> multiple of 8 as IR steps
    (cache_read + pad_block) instead of a device relayout."""
    if spec.transposed or spec.groups != 1 or spec.op == "DEP":
        raise ValueError("direct form: forward convolutions with groups == 1")
    r = spec.spatial_rank
    name = name or spec.op.lower()
    out_sp = spec.out_dhw()[3 - r:]
    in_sp, ks, ss, ps, ds = (t[3 - r:] for t in (spec.in_dhw, spec.k, spec.s, spec.p, spec.d))
    sp = ["d", "h", "w"][3 - r:]
    loops = [("n", spec.n)] + list(zip(sp, out_sp)) + [("co", spec.co)] + [(f"r{s}", k) for s, k in zip(sp, ks)] + \
        [("rc", spec.ci)]
    binds = [f"spatial vn: {spec.n} = n"] + [f"spatial v{s}: {e} = {s}" for s, e in zip(sp, out_sp)] + \
        [f"spatial vco: {spec.co} = co"] + [f"reduce vr{s}: {k} = r{s}" for s, k in zip(sp, ks)] + \
        [f"reduce vrc: {spec.ci} = rc"]
    in_idx, conds = [], []
    for s, I, s_, p_, d_ in zip(sp, in_sp, ss, ps, ds):
        base = f"v{s}" if s_ == 1 else f"v{s}*{s_}"
        tap = f"vr{s}" if d_ == 1 else f"vr{s}*{d_}"
        idx = f"{base} + {tap}" + (f" - {p_}" if p_ else "")
        in_idx.append(idx)
        if p_ > 0:
            conds += [f"{idx} >= 0", f"{idx} < {I}"]
    a_idx = ", ".join(["vn", *in_idx, "vrc"])
    y_idx = ", ".join(["vn", *[f"v{s}" for s in sp], "vco"])
    w_idx = ", ".join([*[f"vr{s}" for s in sp], "vrc", "vco"])
    region = lambda idx: ", ".join(f"{x} +: 1" for x in idx.split(", "))  # noqa: E731
    a_load = f"f32(A[{a_idx}])"
    if conds:
        a_load = f"select({' and '.join(conds)}, {a_load}, 0.0)"
    ind = "    "
    lines = []
    for depth, (v, e) in enumerate(loops):
        lines.append(ind * depth + f"for {v} in 0..{e} {{")
    depth = len(loops)
    body = (f"block conv({', '.join(binds)}) reads(A[{region(a_idx)}], B[{region(w_idx)}]) "
            f"writes(C[{region(y_idx)}]) {{\n  init {{\n    C[{y_idx}] = 0.0\n  }}\n"
            f"  C[{y_idx}] = C[{y_idx}] + {a_load}*f32(B[{w_idx}])\n}}")
    lines += [ind * depth + ln for ln in body.split("\n")]
    for d in range(depth - 1, -1, -1):
        lines.append(ind * d + "}")
    header = (f"func {name}(A: f16[{_dims(None, spec.x_shape())}], B: f16[{_dims(None, spec.w_shape())}], "
              f"C: f32[{_dims(None, spec.y_shape())}]) {{\n  block root() {{\n")
    return header + "\n".join("    " + ln for ln in lines) + "\n  }\n}\n"
