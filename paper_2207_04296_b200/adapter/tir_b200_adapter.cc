// tir_b200_adapter.cc — HostKernel adapter over the C-ABI (see the header).
//
// Packing: TensorView exposes only per-element accessors (interp.h:57-83), so
// the views are packed row-major into host f32 staging (F16 values are f32
// storage in the interpreter, ir.cc:36-47), handed to the synchronous
// host-buffer entry points of include/tir_b200.h (which convert to fp16 on the
// device and reject values fp16 cannot represent), and the accumulated output
// is written back through set_f.
#include "tir_b200_adapter.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "tir/structural.h"
#include "tir/text.h"
#include "tir/validate.h"
#include "tir_b200_tensorize.h"

namespace tir_b200 {
namespace {

std::vector<int64_t> extents_of(const tir::TensorView& v) { return v.extents(); }

int64_t cells_of(const std::vector<int64_t>& e) {
  int64_t n = 1;
  for (int64_t x : e) n *= x;
  return n;
}

// Walks the cells [begin, end) of a row-major view extent, calling f(idx, flat).
template <typename F>
void for_each_index(const std::vector<int64_t>& ext, int64_t begin, int64_t end, F&& f) {
  if (begin >= end) return;
  std::vector<int64_t> idx(ext.size(), 0);
  int64_t rem = begin;
  for (int d = static_cast<int>(ext.size()) - 1; d >= 0; --d) {
    idx[d] = rem % ext[d];
    rem /= ext[d];
  }
  for (int64_t flat = begin; flat < end; ++flat) {
    f(idx, flat);
    int d = static_cast<int>(idx.size()) - 1;
    while (d >= 0 && ++idx[d] == ext[d]) idx[d--] = 0;
  }
}

// TensorView offers only per-element get_f / set_f (interp.h:57-83; no pointer
// accessor by design), at ~50-130 ns a cell. Large views are walked by up to
// 32 threads over disjoint flat ranges: get_f only reads, and set_f of distinct
// cells writes distinct bytes of the tensor's storage, so the ranges never
// touch the same memory.
template <typename F>
void parallel_cells(const std::vector<int64_t>& ext, F&& f) {
  const int64_t n = cells_of(ext);
  if (n == 0) return;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t threads = std::min<int64_t>({static_cast<int64_t>(hw), 32, (n + 65535) / 65536});
  if (threads <= 1) {
    for_each_index(ext, 0, n, f);
    return;
  }
  std::vector<std::thread> pool;
  for (int64_t t = 0; t < threads; ++t)
    pool.emplace_back([&, t] { for_each_index(ext, n * t / threads, n * (t + 1) / threads, f); });
  for (auto& th : pool) th.join();
}

struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double s() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};
thread_local double t_pack = 0, t_device = 0, t_unpack = 0;

std::vector<float> pack(const tir::TensorView& v) {
  Timer t;
  std::vector<float> out(static_cast<size_t>(v.cells()));
  parallel_cells(extents_of(v), [&](const std::vector<int64_t>& idx, int64_t flat) {
    out[static_cast<size_t>(flat)] = static_cast<float>(v.get_f(idx));
  });
  t_pack += t.s();
  return out;
}

void unpack(tir::TensorView& v, const std::vector<float>& data) {
  Timer t;
  parallel_cells(extents_of(v), [&](const std::vector<int64_t>& idx, int64_t flat) {
    v.set_f(idx, data[static_cast<size_t>(flat)]);
  });
  t_unpack += t.s();
}

[[noreturn]] void raise(int rc) {
  const char* kind = rc == TIR_B200_ERR_VALUE         ? "ValueError"
                     : rc == TIR_B200_ERR_UNSUPPORTED ? "UnsupportedShape"
                                                      : "CudaError";
  tir::throw_error(kind, tir_b200_last_error());
}

void require(bool ok, const std::string& msg) {
  if (!ok) tir::throw_error("ValueError", msg);
}

void require_float(const tir::TensorView& v, const char* what) {
  require(tir::dtype_is_float(v.dtype()), std::string(what) + " must be a float view");
}

std::vector<int64_t> conv_x_shape(const tir_b200_conv_desc& d, int rank) {
  const int64_t sp[3] = {d.in_d, d.in_h, d.in_w};
  std::vector<int64_t> s{d.n};
  for (int i = 3 - rank; i < 3; ++i) s.push_back(sp[i]);
  s.push_back(d.ci);
  return s;
}

std::vector<int64_t> conv_w_shape(const tir_b200_conv_desc& d, int rank) {
  const int64_t k[3] = {d.k_d, d.k_h, d.k_w};
  std::vector<int64_t> s;
  for (int i = 3 - rank; i < 3; ++i) s.push_back(k[i]);
  if (d.op != TIR_B200_DEP) s.push_back(d.ci / d.groups);
  s.push_back(d.co);
  return s;
}

std::vector<int64_t> conv_y_shape(const tir_b200_conv_desc& d, int rank) {
  int64_t out[3];
  int rc = tir_b200_conv_out_shape(&d, out);
  if (rc) raise(rc);
  std::vector<int64_t> s{d.n};
  for (int i = 3 - rank; i < 3; ++i) s.push_back(out[i]);
  s.push_back(d.co);
  return s;
}

int conv_rank(const tir_b200_conv_desc& d) {
  return d.op == TIR_B200_C1D ? 1 : d.op == TIR_B200_C3D ? 3 : 2;
}

}  // namespace

void register_gmm(tir::ExecContext& ctx, const std::string& name, bool accumulate) {
  ctx.register_host_kernel(name, [name, accumulate](std::vector<tir::TensorView>& views) {
    require(views.size() == 3, name + ": expects views [C, A, B]");
    tir::TensorView& c = views[0];
    const tir::TensorView& a = views[1];
    const tir::TensorView& b = views[2];
    require_float(c, "C");
    require_float(a, "A");
    require_float(b, "B");
    const auto ce = c.extents(), ae = a.extents(), be = b.extents();
    require(ce.size() == 2 && ae.size() == 2 && be.size() == 2, name + ": operands must be 2-D");
    const int64_t M = ae[0], K = ae[1], N = be[1];
    require(be[0] == K && ce[0] == M && ce[1] == N, name + ": operand extents do not form C[M,N] += A[M,K].B[K,N]");
    std::vector<float> A = pack(a), B = pack(b);
    std::vector<float> C = accumulate ? pack(c) : std::vector<float>(static_cast<size_t>(M * N));
    Timer t;
    int rc = tir_b200_gmm_host_f32(A.data(), B.data(), C.data(), M, N, K, accumulate ? 1 : 0);
    t_device += t.s();
    if (rc) raise(rc);
    unpack(c, C);
  });
}

void register_conv(tir::ExecContext& ctx, const std::string& name, const tir_b200_conv_desc& desc,
                   bool accumulate) {
  // Validate once at registration; geometry errors surface here, not mid-run.
  int64_t out[3];
  int rc = tir_b200_conv_out_shape(&desc, out);
  if (rc) raise(rc);
  ctx.register_host_kernel(name, [name, desc, accumulate](std::vector<tir::TensorView>& views) {
    require(views.size() == 3, name + ": expects views [Y, X, W]");
    tir::TensorView& y = views[0];
    const tir::TensorView& x = views[1];
    const tir::TensorView& w = views[2];
    require_float(y, "Y");
    require_float(x, "X");
    require_float(w, "W");
    const int r = conv_rank(desc);
    require(x.extents() == conv_x_shape(desc, r), name + ": X view does not match the descriptor");
    require(w.extents() == conv_w_shape(desc, r), name + ": W view does not match the descriptor");
    require(y.extents() == conv_y_shape(desc, r), name + ": Y view does not match the descriptor");
    std::vector<float> X = pack(x), W = pack(w);
    std::vector<float> Y = accumulate ? pack(y) : std::vector<float>(static_cast<size_t>(y.cells()));
    Timer t;
    int rc2 = tir_b200_conv_host_f32(&desc, X.data(), W.data(), Y.data(), accumulate ? 1 : 0);
    t_device += t.s();
    if (rc2) raise(rc2);
    unpack(y, Y);
  });
}

std::string conv_intrin_name(const tir_b200_conv_desc& d) {
  static const char* tags[] = {"gmm", "c1d", "c2d", "c3d", "dil", "grp", "t2d", "dep"};
  const char* tag = (d.op >= 0 && d.op <= 7) ? tags[d.op] : "conv";
  return std::string("b200.") + tag + ".s" + std::to_string(d.s_w) + "p" + std::to_string(d.p_w) +
         "d" + std::to_string(d.d_w) + "g" + std::to_string(d.groups);
}

}  // namespace tir_b200

// ---------------------------------------------------------------------------
// C entry points for the drop-in tests (tests/test_dropin.py, ctypes). Errors
// come back as "Kind|message" in `err`.
namespace {

void run_program(const tir::PrimFunc& f, tir::ExecContext& ctx, int n_in, const float* const* inputs,
                 float* out, int64_t out_elems, int64_t* intrinsic_calls) {
  auto in_params = tir::input_params(f);
  if (static_cast<int>(in_params.size()) != n_in) tir::throw_error("ValueError", "input count mismatch");
  std::vector<tir::TensorValue> vals;
  for (int i = 0; i < n_in; ++i) {
    tir::TensorValue t = tir::TensorValue::zeros(in_params[i]->dtype, in_params[i]->shape);
    std::memcpy(t.data.data(), inputs[i], t.data.size());
    vals.push_back(std::move(t));
  }
  auto outs = tir::run(f, vals, ctx);
  if (intrinsic_calls) *intrinsic_calls = ctx.counters.intrinsic_calls;
  if (outs.empty() || outs[0].num_elements() != out_elems)
    tir::throw_error("ValueError", "unexpected output shape");
  std::memcpy(out, outs[0].data.data(), static_cast<size_t>(out_elems) * 4);
}

template <typename F>
int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const tir::Error& e) {
    std::snprintf(err, static_cast<size_t>(errlen), "%s|%s", e.kind().c_str(), e.message().c_str());
  } catch (const std::exception& e) {
    std::snprintf(err, static_cast<size_t>(errlen), "InternalError|%s", e.what());
  }
  return -1;
}

void copy_out(const std::string& s, char* dst, int64_t len, const char* what) {
  if (!dst) return;
  if (static_cast<int64_t>(s.size()) + 1 > len) tir::throw_error("ValueError", std::string(what) + " buffer too small");
  std::memcpy(dst, s.c_str(), s.size() + 1);
}

}  // namespace

// Parse a program, register the B200 intrinsic on a fresh ExecContext and run
// the reference interpreter, which dispatches every tensorized block to the
// GPU through the HostKernels above.
extern "C" int tir_b200_adapter_run(const char* ir_text, const char* intrin,
                                    const tir_b200_conv_desc* desc, int n_in,
                                    const float* const* inputs, float* out, int64_t out_elems,
                                    int64_t* intrinsic_calls, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    tir::PrimFuncPtr f = tir::parse_text(ir_text);
    tir::ExecContext ctx;
    if (desc) {
      tir_b200::register_conv(ctx, intrin, *desc);
    } else {
      tir_b200::register_gmm(ctx, intrin);
    }
    run_program(*f, ctx, n_in, inputs, out, out_elems, intrinsic_calls);
  });
}

// The tensorize composite on `block` of a scalar program: returns the rewritten
// program text, its trace (JSONL), the generated intrinsic name and the match
// (desc->op == TIR_B200_GMM with mnk for GMM). Also checks that the result is
// validate_all-clean and that replaying the trace on a fresh parse of the
// source reproduces it structurally (ValidationFailed / ReplayMismatch).
extern "C" int tir_b200_adapter_tensorize(const char* ir_text, const char* block, char* text, int64_t text_len,
                                          char* trace, int64_t trace_len, char* intrin, int64_t intrin_len,
                                          tir_b200_conv_desc* desc, int64_t* mnk, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    tir_b200::register_tensorize_step_handler();
    tir::Schedule s(tir::parse_text(ir_text));
    tir_b200::OpMatch m = tir_b200::tensorize_whole_op(s, block);
    auto diags = tir::validate_all(*s.func());
    if (tir::has_errors(diags)) tir::throw_error("ValidationFailed", tir::format_diagnostic(diags.front()));
    tir::Schedule again = tir::replay(s.trace(), tir::parse_text(ir_text));
    if (!tir::structural_equal(*again.func(), *s.func())) tir::throw_error("ReplayMismatch", "trace replay differs");
    copy_out(tir::print_text(s.func()), text, text_len, "text");
    copy_out(tir::trace_to_jsonl(s.trace()), trace, trace_len, "trace");
    copy_out(m.intrin, intrin, intrin_len, "intrin");
    if (desc) {
      *desc = m.conv;
      if (m.gmm) desc->op = TIR_B200_GMM;
    }
    if (mnk) {
      mnk[0] = m.m;
      mnk[1] = m.n;
      mnk[2] = m.k;
    }
  });
}

// Tensorize each named block of a scalar program, register the matched B200
// kernels and run it through tir::run (blocks not named stay scalar).
extern "C" int tir_b200_adapter_run_auto(const char* ir_text, const char* const* blocks, int n_blocks, int n_in,
                                         const float* const* inputs, float* out, int64_t out_elems,
                                         int64_t* intrinsic_calls, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    tir::Schedule s(tir::parse_text(ir_text));
    tir::ExecContext ctx;
    for (int i = 0; i < n_blocks; ++i) tir_b200::register_matched(ctx, tir_b200::tensorize_whole_op(s, blocks[i]));
    run_program(*s.func(), ctx, n_in, inputs, out, out_elems, intrinsic_calls);
  });
}

// Channel pad as IR steps (tir_b200_tensorize.h, pad_conv_channels): returns the
// rewritten program and its trace (JSONL), after checking that replaying the trace
// on a fresh parse reproduces it.
extern "C" int tir_b200_adapter_pad_channels(const char* ir_text, const char* block, int64_t multiple, char* text,
                                             int64_t text_len, char* trace, int64_t trace_len, int64_t* padded,
                                             char* err, int errlen) {
  return guarded(err, errlen, [&] {
    tir::Schedule s(tir::parse_text(ir_text));
    const int64_t p = tir_b200::pad_conv_channels(s, block, multiple);
    tir::Schedule again = tir::replay(s.trace(), tir::parse_text(ir_text));
    if (!tir::structural_equal(*again.func(), *s.func())) tir::throw_error("ReplayMismatch", "trace replay differs");
    copy_out(tir::print_text(s.func()), text, text_len, "text");
    copy_out(tir::trace_to_jsonl(s.trace()), trace, trace_len, "trace");
    if (padded) *padded = p;
  });
}

// Drop-in end-to-end timing (bench.py e2e_interp): tensorize `block` of a scalar
// program once, then time `runs` complete tir::run calls — the reference's own
// interpreter dispatching the tensorized block to the B200 kernel through the
// HostKernel above (view packing, host-buffer C-ABI call with its H2D / D2H,
// write-back). Returns seconds per run and its split (pack / device call /
// unpack) per run; the last run's output goes to `out`.
extern "C" int tir_b200_adapter_time_run(const char* ir_text, const char* block, int n_in,
                                         const float* const* inputs, float* out, int64_t out_elems, int runs,
                                         double* sec_per_run, double* split3, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    tir::Schedule s(tir::parse_text(ir_text));
    tir::ExecContext ctx;
    const tir_b200::OpMatch m = tir_b200::tensorize_whole_op(s, block);
    tir_b200::register_matched(ctx, m);
    run_program(*s.func(), ctx, n_in, inputs, out, out_elems, nullptr);  // warm-up (allocations)
    tir_b200::t_pack = tir_b200::t_device = tir_b200::t_unpack = 0;
    tir_b200::Timer t;
    for (int i = 0; i < runs; ++i) {
      tir::ExecContext c2;
      tir_b200::register_matched(c2, m);
      run_program(*s.func(), c2, n_in, inputs, out, out_elems, nullptr);
    }
    const double total = t.s();
    *sec_per_run = total / runs;
    if (split3) {
      split3[0] = tir_b200::t_pack / runs;
      split3[1] = tir_b200::t_device / runs;
      split3[2] = tir_b200::t_unpack / runs;
    }
  });
}

// SURVEY §8(c) per-intrinsic oracle: the same tensorized program run with the
// reference's OWN scalar implementation of the intrinsic — make_scalar_kernel
// (src/interp.cc:594-726) built from a description PrimFunc `desc_text` (its
// compute block's body, iterated over the block domain; no init: accumulate
// semantics) — registered under the intrinsic's name instead of the B200
// kernel. `params_csv` names the description params in view order
// ("C,A,B": writes[0] first, then reads, interp.cc:371-373).
extern "C" int tir_b200_adapter_run_scalar(const char* ir_text, const char* intrin, const char* desc_text,
                                           const char* params_csv, int n_in, const float* const* inputs, float* out,
                                           int64_t out_elems, int64_t* intrinsic_calls, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<std::string> params;
    std::string cur;
    for (const char* c = params_csv; *c; ++c) {
      if (*c == ',') {
        params.push_back(cur);
        cur.clear();
      } else {
        cur += *c;
      }
    }
    if (!cur.empty()) params.push_back(cur);
    tir::PrimFuncPtr f = tir::parse_text(ir_text);
    tir::ExecContext ctx;
    ctx.register_host_kernel(intrin, tir::make_scalar_kernel(tir::parse_text(desc_text), params));
    run_program(*f, ctx, n_in, inputs, out, out_elems, intrinsic_calls);
  });
}

namespace {

// Names of the views a tensorized block hands its kernel: writes[0], then reads.
std::vector<std::string> operand_names(const tir::PrimFunc& f, const std::string& intrin) {
  std::vector<std::string> names;
  tir::pre_order_stmts(f.body, [&](const tir::Stmt& s) {
    if (s->kind == tir::StmtKind::BlockRealize && s->block) {
      auto it = s->block->annotations.find("tensorized");
      if (it != s->block->annotations.end() && it->second == intrin && names.empty()) {
        names.push_back(s->block->writes.at(0).buffer->name);
        for (const auto& r : s->block->reads) names.push_back(r.buffer->name);
      }
    }
    return names.empty();
  });
  return names;
}

}  // namespace

// Tensorize `block`, then emit a program in the reference grammar: the `intrin`
// declaration of the generated intrinsic (tir_b200_tensorize.h intrin_decl_text)
// followed by the tensorized function. The text is checked to parse back with
// tir::parse_program (one function, one declaration with one constraint per
// view) before it is returned.
extern "C" int tir_b200_adapter_declare(const char* ir_text, const char* block, char* program, int64_t program_len,
                                        char* err, int errlen) {
  return guarded(err, errlen, [&] {
    tir::Schedule s(tir::parse_text(ir_text));
    const tir_b200::OpMatch m = tir_b200::tensorize_whole_op(s, block);
    const auto ops = operand_names(*s.func(), m.intrin);
    const std::string text = tir_b200::intrin_decl_text(m, ops) + "\n" + tir::print_text(s.func());
    tir::ParsedProgram pp = tir::parse_program(text);
    if (pp.funcs.size() != 1 || pp.intrins.size() != 1 || pp.intrins[0].name != m.intrin ||
        pp.intrins[0].constraints.size() != ops.size())
      tir::throw_error("InternalError", "declaration does not round-trip through parse_program");
    copy_out(text, program, program_len, "program");
  });
}

// Run a program whose b200.* intrinsics are registered from its own `intrin`
// declarations (register_declared): no other registration step.
extern "C" int tir_b200_adapter_run_declared(const char* program_text, int n_in, const float* const* inputs,
                                             float* out, int64_t out_elems, int64_t* intrinsic_calls, char* err,
                                             int errlen) {
  return guarded(err, errlen, [&] {
    tir::ParsedProgram pp = tir::parse_program(program_text);
    if (pp.funcs.empty()) tir::throw_error("ValueError", "program has no function");
    tir::ExecContext ctx;
    if (tir_b200::register_declared(ctx, pp) == 0) tir::throw_error("ValueError", "no b200 intrinsic declared");
    run_program(*pp.funcs[0], ctx, n_in, inputs, out, out_elems, intrinsic_calls);
  });
}
