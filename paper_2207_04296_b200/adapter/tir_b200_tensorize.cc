// tir_b200_tensorize.cc — whole-op tensorize composite (see the header).
#include "tir_b200_tensorize.h"

#include <cstdio>
#include <cstring>

#include <algorithm>
#include <map>
#include <set>

#include "tir/analysis.h"
#include "tir/structural.h"
#include "tir/text.h"
#include "tir_b200_adapter.h"

namespace tir_b200 {
namespace {

using tir::Expr;
using tir::ExprKind;
using tir::Stmt;
using tir::StmtKind;

[[noreturn]] void mismatch(const std::string& why) { tir::throw_error("DescMismatch", why); }

Expr strip_cast(Expr e) {
  while (e && e->kind == ExprKind::Cast) e = e->args[0];
  return e;
}

bool is_zero(const Expr& e0) {
  Expr e = strip_cast(e0);
  return e && ((e->kind == ExprKind::FloatConst && e->float_value == 0.0) ||
               (e->kind == ExprKind::IntConst && e->int_value == 0));
}

std::string var_name(const Expr& e) { return e && e->kind == ExprKind::Var ? e->name : std::string(); }

// One multiplicand: a buffer load, optionally under select(cond, load, 0.0)
// (zero padding, SURVEY §8(a) "Padding").
struct Operand {
  tir::BufferPtr buf;
  std::vector<Expr> idx;
  Expr cond;
};

Operand operand_of(const Expr& e0) {
  Expr e = strip_cast(e0);
  Operand op;
  if (e && e->kind == ExprKind::Select) {
    if (!is_zero(e->args[2])) mismatch("select must yield 0.0 when out of bounds");
    op.cond = e->args[0];
    e = strip_cast(e->args[1]);
  }
  if (!e || e->kind != ExprKind::BufferLoad) mismatch("multiplicand is not a buffer load");
  op.buf = e->buffer;
  op.idx = e->args;
  return op;
}

Stmt find_realize(const tir::PrimFunc& f, const std::string& name) {
  Stmt found;
  tir::pre_order_stmts(f.body, [&](const Stmt& s) {
    if (s->kind == StmtKind::BlockRealize && s->block && s->block->name == name) found = s;
    return !found;
  });
  if (!found) tir::throw_error("StaleHandle", "no block named '" + name + "'");
  return found;
}

void conjuncts(const Expr& e, std::vector<Expr>* out) {
  if (!e) return;
  if (e->kind == ExprKind::And) {
    conjuncts(e->args[0], out);
    conjuncts(e->args[1], out);
  } else {
    out->push_back(e);
  }
}

bool const_of(const Expr& e, int64_t* v) { return tir::as_const_int(strip_cast(e), v); }

struct IterInfo {
  int64_t extent = 0;
  tir::IterKind kind = tir::IterKind::DataParallel;
};

// Coefficient of Var `name` among linear terms (0 if absent); every atom must be
// one of the allowed vars.
bool affine_in(const Expr& e, const std::set<std::string>& allowed, std::map<std::string, int64_t>* coeff,
               int64_t* constant) {
  auto terms = tir::linear_terms(e, constant);
  for (const auto& t : terms) {
    const std::string v = var_name(t.atom);
    if (v.empty() || !allowed.count(v)) return false;
    (*coeff)[v] += t.coeff;
  }
  return true;
}

void fill_geometry(tir_b200_conv_desc& d, int r, const std::vector<int64_t>& in, const std::vector<int64_t>& k,
                   const std::vector<int64_t>& s, const std::vector<int64_t>& p, const std::vector<int64_t>& dil) {
  int64_t* in3[3] = {&d.in_d, &d.in_h, &d.in_w};
  int64_t* k3[3] = {&d.k_d, &d.k_h, &d.k_w};
  int64_t* s3[3] = {&d.s_d, &d.s_h, &d.s_w};
  int64_t* p3[3] = {&d.p_d, &d.p_h, &d.p_w};
  int64_t* d3[3] = {&d.d_d, &d.d_h, &d.d_w};
  for (int i = 0; i < 3; ++i) {
    *in3[i] = 1; *k3[i] = 1; *s3[i] = 1; *p3[i] = 0; *d3[i] = 1;
  }
  for (int i = 0; i < r; ++i) {
    const int j = 3 - r + i;
    *in3[j] = in[i]; *k3[j] = k[i]; *s3[j] = s[i]; *p3[j] = p[i]; *d3[j] = dil[i];
  }
}

Stmt rewrite(const Stmt& s, const tir::StmtNode* target, const Stmt& repl) {
  if (!s) return s;
  if (s.get() == target) return repl;
  switch (s->kind) {
    case StmtKind::For: {
      Stmt b = rewrite(s->body, target, repl);
      if (b == s->body) return s;
      auto n = std::make_shared<tir::StmtNode>(*s);
      n->body = b;
      return n;
    }
    case StmtKind::Seq: {
      std::vector<Stmt> v;
      bool changed = false;
      for (const auto& c : s->stmts) {
        v.push_back(rewrite(c, target, repl));
        changed |= v.back() != c;
      }
      if (!changed) return s;
      auto n = std::make_shared<tir::StmtNode>(*s);
      n->stmts = std::move(v);
      return n;
    }
    case StmtKind::BlockRealize: {
      Stmt b = rewrite(s->block->body, target, repl);
      Stmt i = rewrite(s->block->init, target, repl);
      if (b == s->block->body && i == s->block->init) return s;
      auto blk = std::make_shared<tir::Block>(*s->block);
      blk->body = b;
      blk->init = i;
      auto n = std::make_shared<tir::StmtNode>(*s);
      n->block = blk;
      return n;
    }
    default:
      return s;
  }
}

// The step "b200.tensorize": outer block body := intrin(), attrs("tensorized" = intrin).
// drop_init: the outer block's init (the zero store blockize moved out of the
// contraction, schedule_block.cc:570-603) is removed and the call overwrites
// its output instead — for a whole-op block the init would run exactly once,
// right before the single call, so the result is unchanged, while the
// interpreter no longer zero-fills the output element by element and the
// HostKernel neither packs nor uploads it.
void replace_with_call(tir::Schedule& s, const std::string& block, const std::string& intrin, bool drop_init) {
  Stmt o = s.find_block_realize(block);
  if (!o) tir::throw_error("StaleHandle", "no block named '" + block + "'");
  auto blk = std::make_shared<tir::Block>(*o->block);
  blk->body = tir::make_evaluate(tir::make_call(intrin));
  if (drop_init) blk->init = nullptr;
  blk->annotations["tensorized"] = intrin;
  Stmt repl = tir::make_block_realize(o->bindings, o->predicate, blk);
  Stmt body = rewrite(s.func()->body, o.get(), repl);
  tir::TraceStep step;
  step.prim = "b200.tensorize";
  step.args = {{"block", block}, {"intrin", intrin}, {"drop_init", drop_init}};
  s.commit_rewrite(tir::make_func(s.func()->name, s.func()->params, body), std::move(step));
}

}  // namespace

std::string conv_intrin_key(const tir_b200_conv_desc& d) {
  static const char* tags[] = {"gmm", "c1d", "c2d", "c3d", "dil", "grp", "t2d", "dep"};
  const char* tag = (d.op >= 0 && d.op <= 7) ? tags[d.op] : "conv";
  auto x3 = [](int64_t a, int64_t b, int64_t c) {
    return std::to_string(a) + "x" + std::to_string(b) + "x" + std::to_string(c);
  };
  return std::string("b200.") + tag + ".n" + std::to_string(d.n) + "_i" + x3(d.in_d, d.in_h, d.in_w) + "_c" +
         std::to_string(d.ci) + "_o" + std::to_string(d.co) + "_k" + x3(d.k_d, d.k_h, d.k_w) + "_s" +
         x3(d.s_d, d.s_h, d.s_w) + "_p" + x3(d.p_d, d.p_h, d.p_w) + "_d" + x3(d.d_d, d.d_h, d.d_w) + "_g" +
         std::to_string(d.groups);
}

OpMatch match_contraction(const tir::PrimFunc& f, const std::string& block) {
  Stmt realize = find_realize(f, block);
  const tir::Block& B = *realize->block;
  if (B.annotations.count("tensorized")) mismatch("block '" + block + "' is already tensorized");
  // A guarded block (a `where` predicate, e.g. from a padded split) writes only
  // part of its domain; the whole-op kernels write every output element.
  if (realize->predicate && !tir::is_true(realize->predicate))
    mismatch("block '" + block + "' has a predicate; whole-op kernels cannot honour it");
  std::map<std::string, IterInfo> iters;
  for (const auto& iv : B.iter_vars) {
    IterInfo info;
    int64_t lo = 0;
    if (!tir::as_const_int(iv.domain.min, &lo) || lo != 0 || !tir::as_const_int(iv.domain.extent, &info.extent))
      mismatch("iterator domains must be constant and zero-based");
    info.kind = iv.kind;
    iters[var_name(iv.var)] = info;
  }
  auto is_iter = [&](const std::string& v, tir::IterKind k) {
    auto it = iters.find(v);
    return it != iters.end() && it->second.kind == k;
  };
  auto ext = [&](const std::string& v) { return iters.at(v).extent; };

  // body: Y[ys] = Y[ys] + a * b
  const Stmt& st = B.body;
  if (!st || st->kind != StmtKind::BufferStore) mismatch("block body must be a single buffer store");
  const tir::BufferPtr Y = st->buffer;
  if (Y->dtype != tir::DType::F32) mismatch("output must be f32 (fp32 accumulation)");
  std::vector<std::string> ys;
  for (const auto& e : st->indices) {
    const std::string v = var_name(e);
    if (!is_iter(v, tir::IterKind::DataParallel)) mismatch("output indices must be spatial iterators");
    ys.push_back(v);
  }
  if (std::set<std::string>(ys.begin(), ys.end()).size() != ys.size()) mismatch("repeated output iterator");
  const Expr& val = st->value;
  if (!val || val->kind != ExprKind::Add) mismatch("update must be Y = Y + a*b");
  auto is_self = [&](const Expr& e) {
    if (!e || e->kind != ExprKind::BufferLoad || e->buffer->name != Y->name || e->args.size() != ys.size())
      return false;
    for (size_t i = 0; i < ys.size(); ++i)
      if (var_name(e->args[i]) != ys[i]) return false;
    return true;
  };
  Expr prod;
  if (is_self(val->args[0])) prod = val->args[1];
  else if (is_self(val->args[1])) prod = val->args[0];
  else mismatch("update must accumulate into the stored element");
  prod = strip_cast(prod);
  if (!prod || prod->kind != ExprKind::Mul) mismatch("update must add a product");
  Operand a = operand_of(prod->args[0]), b = operand_of(prod->args[1]);
  for (const Operand* o : {&a, &b})
    if (!tir::dtype_is_float(o->buf->dtype)) mismatch("operands must be float (f16 values)");
  // X is the operand indexed by the leading output iterator (M for GMM, batch for conv)
  auto leads = [&](const Operand& o) { return !o.idx.empty() && var_name(o.idx[0]) == ys[0]; };
  if (leads(a) == leads(b)) mismatch("cannot tell the input from the weights");
  const Operand& X = leads(a) ? a : b;
  const Operand& W = leads(a) ? b : a;
  if (W.cond) mismatch("weights must not be guarded");
  if (B.init) {
    const Stmt& in = B.init;
    if (in->kind != StmtKind::BufferStore || in->buffer->name != Y->name || !is_zero(in->value))
      mismatch("init must be Y = 0.0");
  }
  for (const auto& [v, info] : iters) {
    bool used = std::find(ys.begin(), ys.end(), v) != ys.end();
    for (const auto& e : W.idx) used |= var_name(e) == v;
    std::set<std::string> fv;
    for (const auto& e : X.idx) tir::collect_free_vars(e, &fv);
    used |= fv.count(v) > 0;
    if (!used && info.extent != 1) mismatch("iterator '" + v + "' is unused by the contraction");
  }

  OpMatch m;
  m.overwrite = B.init != nullptr;  // Y = 0 (checked above), then Y += ...: the call may overwrite
  const size_t R = ys.size();
  if (R == 2) {  // GMM: Y[i, j] += X[i, k] * W[k, j]
    const std::string vk = X.idx.size() == 2 ? var_name(X.idx[1]) : "";
    if (X.cond || X.idx.size() != 2 || W.idx.size() != 2 || !is_iter(vk, tir::IterKind::Reduction) ||
        var_name(W.idx[0]) != vk || var_name(W.idx[1]) != ys[1])
      mismatch("rank-2 output but not C[i,j] += A[i,k]*B[k,j]");
    m.gmm = true;
    m.m = ext(ys[0]);
    m.n = ext(ys[1]);
    m.k = ext(vk);
    if (Y->shape != std::vector<int64_t>{m.m, m.n} || X.buf->shape != std::vector<int64_t>{m.m, m.k} ||
        W.buf->shape != std::vector<int64_t>{m.k, m.n})
      mismatch("GMM iterator extents do not cover the buffers (not a whole-op block)");
    m.intrin = m.overwrite ? "b200.gmm.ow" : "b200.gmm";
    return m;
  }
  if (R < 3 || R > 5) mismatch("unsupported output rank");
  const int r = static_cast<int>(R) - 2;
  const std::string vn = ys[0], vco = ys[R - 1];
  if (X.idx.size() != R) mismatch("input rank does not match the output");
  const bool dep = W.idx.size() == static_cast<size_t>(r) + 1;
  if (!dep && W.idx.size() != static_cast<size_t>(r) + 2) mismatch("weight rank");
  std::vector<std::string> vr(r);
  for (int i = 0; i < r; ++i) {
    vr[i] = var_name(W.idx[i]);
    if (!is_iter(vr[i], tir::IterKind::Reduction)) mismatch("weight taps must be reduction iterators");
  }
  if (var_name(W.idx.back()) != vco) mismatch("weights must be indexed by the output channel last");
  const int64_t N = ext(vn), CO = ext(vco);
  int64_t CI = 0, G = 1, cig = 1;
  const Expr& chan = X.idx.back();
  if (dep) {
    if (var_name(chan) != vco) mismatch("depthwise input channel must be the output channel");
    CI = CO;
    G = CO;
  } else {
    const std::string vrc = var_name(W.idx[r]);
    if (!is_iter(vrc, tir::IterKind::Reduction)) mismatch("weight input channel must be a reduction iterator");
    cig = ext(vrc);
    if (var_name(chan) == vrc) {
      G = 1;
    } else {  // grouped: (vco / cog) * cig + vrc
      int64_t c0 = 0;
      auto terms = tir::linear_terms(chan, &c0);
      int64_t cog = 0, coeff = 0;
      bool has_rc = false;
      for (const auto& t : terms) {
        if (var_name(t.atom) == vrc && t.coeff == 1) {
          has_rc = true;
        } else if (t.atom->kind == ExprKind::FloorDiv && var_name(t.atom->args[0]) == vco &&
                   const_of(t.atom->args[1], &cog)) {
          coeff = t.coeff;
        } else {
          mismatch("input channel expression is not (co / (CO/G)) * (CI/G) + rc");
        }
      }
      if (c0 != 0 || !has_rc || cog <= 0 || CO % cog || coeff != cig) mismatch("bad group channel map");
      G = CO / cog;
    }
    CI = G * cig;
  }
  // spatial dims: forward  x = o*s + k*d - p ;  transposed  x = (o + p - k*d) / s
  std::vector<int64_t> I(r), K(r), S(r), P(r), D(r), O(r);
  std::vector<Expr> xidx(r), tnum(r);
  int transposed = -1;
  for (int i = 0; i < r; ++i) {
    const std::string vo = ys[1 + i];
    O[i] = ext(vo);
    K[i] = ext(vr[i]);
    I[i] = X.buf->shape[1 + i];
    xidx[i] = X.idx[1 + i];
    Expr t = xidx[i];
    int64_t s = 1;
    bool div = false;
    if (t->kind == ExprKind::FloorDiv) {
      if (!const_of(t->args[1], &s) || s < 1) mismatch("transposed stride must be a constant");
      t = t->args[0];
      div = true;
    }
    tnum[i] = t;
    std::map<std::string, int64_t> c;
    int64_t c0 = 0;
    if (!affine_in(t, {vo, vr[i]}, &c, &c0)) mismatch("input index is not affine in (output, tap)");
    const int64_t co_ = c[vo], cr = c[vr[i]];
    const bool tr = div || cr < 0;
    if (transposed >= 0 && transposed != static_cast<int>(tr)) mismatch("mixed forward/transposed dims");
    transposed = tr;
    if (tr) {
      if (co_ != 1 && O[i] != 1) mismatch("transposed index must be (o + p - k*d) / s");
      if (cr == 0 && K[i] != 1) mismatch("input index ignores an iterator");
      S[i] = s;
      D[i] = cr == 0 ? 1 : -cr;
      P[i] = c0;
    } else {
      S[i] = co_ == 0 ? 1 : co_;
      D[i] = cr == 0 ? 1 : cr;
      P[i] = -c0;
      if ((co_ == 0 && O[i] != 1) || (cr == 0 && K[i] != 1)) mismatch("input index ignores an iterator");
    }
    if (S[i] < 1 || D[i] < 1 || P[i] < 0) mismatch("stride, dilation and padding must be non-negative");
  }
  // guards: each conjunct must be a bounds / parity test of an input index
  std::vector<Expr> conds;
  conjuncts(X.cond, &conds);
  std::vector<bool> lo(r, false), hi(r, false), par(r, false);
  for (const auto& e : conds) {
    bool ok = false;
    for (int i = 0; i < r && !ok; ++i) {
      int64_t v = 0;
      const auto& a0 = e->args.size() > 0 ? e->args[0] : Expr();
      const auto& a1 = e->args.size() > 1 ? e->args[1] : Expr();
      auto same = [&](const Expr& x, const Expr& y) { return x && y && tir::structural_equal(x, y); };
      if ((e->kind == ExprKind::Ge && same(a0, xidx[i]) && const_of(a1, &v) && v == 0) ||
          (e->kind == ExprKind::Le && same(a1, xidx[i]) && const_of(a0, &v) && v == 0)) {
        lo[i] = ok = true;
      } else if ((e->kind == ExprKind::Lt && same(a0, xidx[i]) && const_of(a1, &v) && v == I[i]) ||
                 (e->kind == ExprKind::Gt && same(a1, xidx[i]) && const_of(a0, &v) && v == I[i])) {
        hi[i] = ok = true;
      } else if (e->kind == ExprKind::Eq && a0 && a0->kind == ExprKind::FloorMod && same(a0->args[0], tnum[i]) &&
                 const_of(a0->args[1], &v) && v == S[i] && const_of(a1, &v) && v == 0) {
        par[i] = ok = true;
      }
    }
    if (!ok) mismatch("unrecognised guard '" + tir::print_expr(e) + "'");
  }
  for (int i = 0; i < r; ++i) {
    bool need_lo, need_hi, need_par = false;
    if (transposed) {
      need_lo = P[i] - (K[i] - 1) * D[i] < 0;
      need_hi = (O[i] - 1 + P[i]) / S[i] > I[i] - 1;
      need_par = S[i] > 1;
    } else {
      need_lo = P[i] > 0;
      need_hi = (O[i] - 1) * S[i] + (K[i] - 1) * D[i] - P[i] > I[i] - 1;
    }
    if ((need_lo && !lo[i]) || (need_hi && !hi[i]) || (need_par && !par[i]))
      mismatch("input index can leave the tensor without a select guard");
  }
  tir_b200_conv_desc d{};
  d.transposed = transposed ? 1 : 0;
  d.n = N;
  d.ci = CI;
  d.co = CO;
  d.groups = G;
  fill_geometry(d, r, I, K, S, P, D);
  bool dil = false;
  for (int i = 0; i < r; ++i) dil |= D[i] != 1;
  d.op = dep ? TIR_B200_DEP
             : transposed ? TIR_B200_T2D
             : r == 1     ? TIR_B200_C1D
             : r == 3     ? TIR_B200_C3D
             : G > 1      ? TIR_B200_GRP
             : dil        ? TIR_B200_DIL
                          : TIR_B200_C2D;
  int64_t out[3];
  if (tir_b200_conv_out_shape(&d, out) != TIR_B200_OK) mismatch(std::string("geometry: ") + tir_b200_last_error());
  for (int i = 0; i < r; ++i)
    if (out[3 - r + i] != O[i]) mismatch("output extent does not match the conv geometry");
  // whole-op: iterator extents equal the buffers
  std::vector<int64_t> xs{N}, ws, yshape{N};
  for (int i = 0; i < r; ++i) {
    xs.push_back(I[i]);
    ws.push_back(K[i]);
    yshape.push_back(O[i]);
  }
  xs.push_back(CI);
  if (!dep) ws.push_back(cig);
  ws.push_back(CO);
  yshape.push_back(CO);
  if (X.buf->shape != xs || W.buf->shape != ws || Y->shape != yshape)
    mismatch("conv iterator extents do not cover the buffers (not a whole-op block)");
  m.conv = d;
  m.intrin = conv_intrin_key(d) + (m.overwrite ? ".ow" : "");
  return m;
}

OpMatch tensorize_whole_op(tir::Schedule& s, const std::string& block) {
  OpMatch m = match_contraction(*s.func(), block);
  tir::Schedule trial = s;
  auto loops = trial.loops_of(block);
  if (loops.empty()) tir::throw_error("NotWholeOp", "block '" + block + "' has no enclosing loop");
  const std::string outer = trial.blockize(loops.front());
  Stmt o = trial.find_block_realize(outer);
  for (size_t i = 0; i < o->block->iter_vars.size(); ++i) {
    int64_t e = 0;
    if (!tir::as_const_int(o->block->iter_vars[i].domain.extent, &e) || e != 1 ||
        !tir::is_const_int(o->bindings[i], 0))
      tir::throw_error("NotWholeOp", "the loop nest of '" + block + "' covers only part of the op");
  }
  replace_with_call(trial, outer, m.intrin, m.overwrite);
  s = trial;
  return m;
}

std::string intrin_decl_text(const OpMatch& m, const std::vector<std::string>& operands) {
  std::string t = "intrin " + m.intrin + " {\n";
  for (const auto& o : operands) t += "  require " + o + " scope(\"global\") contiguous\n";
  return t + "}\n";
}

OpMatch decode_intrin(const std::string& name) {
  OpMatch m;
  std::string key = name;
  if (key.size() > 3 && key.compare(key.size() - 3, 3, ".ow") == 0) {
    m.overwrite = true;
    key.resize(key.size() - 3);
  }
  m.intrin = name;
  if (key == "b200.gmm") {
    m.gmm = true;
    return m;
  }
  static const char* tags[] = {"gmm", "c1d", "c2d", "c3d", "dil", "grp", "t2d", "dep"};
  tir_b200_conv_desc d{};
  char tag[8] = {0};
  long long v[20];
  const int got = std::sscanf(key.c_str(),
                              "b200.%7[a-z0-9].n%lld_i%lldx%lldx%lld_c%lld_o%lld_k%lldx%lldx%lld_s%lldx%lldx%lld_p%lldx%lldx"
                              "%lld_d%lldx%lldx%lld_g%lld",
                              tag, &v[0], &v[1], &v[2], &v[3], &v[4], &v[5], &v[6], &v[7], &v[8], &v[9], &v[10],
                              &v[11], &v[12], &v[13], &v[14], &v[15], &v[16], &v[17], &v[18]);
  if (got != 20) tir::throw_error("DescMismatch", "'" + name + "' is not a b200 intrinsic name");
  d.op = -1;
  for (int i = 0; i < 8; ++i)
    if (!std::strcmp(tag, tags[i])) d.op = i;
  if (d.op <= 0) tir::throw_error("DescMismatch", "'" + name + "': unknown operator tag");
  d.transposed = d.op == TIR_B200_T2D;
  d.n = v[0];
  d.in_d = v[1]; d.in_h = v[2]; d.in_w = v[3];
  d.ci = v[4]; d.co = v[5];
  d.k_d = v[6]; d.k_h = v[7]; d.k_w = v[8];
  d.s_d = v[9]; d.s_h = v[10]; d.s_w = v[11];
  d.p_d = v[12]; d.p_h = v[13]; d.p_w = v[14];
  d.d_d = v[15]; d.d_h = v[16]; d.d_w = v[17];
  d.groups = v[18];
  if (conv_intrin_key(d) != key) tir::throw_error("DescMismatch", "'" + name + "' does not round-trip");
  int64_t out[3];
  if (tir_b200_conv_out_shape(&d, out) != TIR_B200_OK)
    tir::throw_error("DescMismatch", "'" + name + "': " + tir_b200_last_error());
  m.conv = d;
  return m;
}

int register_declared(tir::ExecContext& ctx, const tir::ParsedProgram& program) {
  int n = 0;
  for (const auto& decl : program.intrins) {
    if (decl.name.rfind("b200.", 0) != 0) continue;  // someone else's intrinsic
    if (!decl.exec_scope.empty())
      tir::throw_error("DescMismatch", decl.name + ": B200 whole-op intrinsics take no exec_scope");
    for (const auto& [param, c] : decl.constraints)
      if (!c.scope.empty() && c.scope != "global")
        tir::throw_error("DescMismatch", decl.name + ": operand " + param + " must be in global scope");
    register_matched(ctx, decode_intrin(decl.name));
    ++n;
  }
  return n;
}

void register_matched(tir::ExecContext& ctx, const OpMatch& m) {
  if (ctx.has_kernel(m.intrin)) return;
  if (m.gmm) {
    register_gmm(ctx, m.intrin, !m.overwrite);
  } else {
    register_conv(ctx, m.intrin, m.conv, !m.overwrite);
  }
}

namespace {

void widen_reads(tir::Schedule& s, const std::string& block) {
  Stmt o = s.find_block_realize(block);
  if (!o) tir::throw_error("StaleHandle", "no block named '" + block + "'");
  auto blk = std::make_shared<tir::Block>(*o->block);
  for (auto& r : blk->reads) {
    r.ranges.clear();
    for (int64_t d : r.buffer->shape) r.ranges.push_back(tir::const_range(0, d));
  }
  Stmt repl = tir::make_block_realize(o->bindings, o->predicate, blk);
  Stmt body = rewrite(s.func()->body, o.get(), repl);
  tir::TraceStep step;
  step.prim = "b200.widen_reads";
  step.args = {{"block", block}};
  s.commit_rewrite(tir::make_func(s.func()->name, s.func()->params, body), std::move(step));
}

void register_widen_handler() {
  static const bool registered = [] {
    tir::register_step_handler("b200.widen_reads", [](tir::Schedule& s, const tir::TraceStep& step) {
      widen_reads(s, step.args.at("block").get<std::string>());
    });
    return true;
  }();
  (void)registered;
}

}  // namespace

int64_t pad_conv_channels(tir::Schedule& s, const std::string& block, int64_t multiple) {
  register_widen_handler();
  Stmt realize = s.find_block_realize(block);
  if (!realize) tir::throw_error("StaleHandle", "no block named '" + block + "'");
  const auto& ivs = realize->block->iter_vars;
  std::vector<int64_t> ext(ivs.size());
  int64_t padded = -1;
  for (size_t i = 0; i < ivs.size(); ++i) {
    if (!tir::as_const_int(ivs[i].domain.extent, &ext[i])) tir::throw_error("NotSchedulable", "non-constant domain");
    if (var_name(ivs[i].var) == "vrc") {
      padded = (ext[i] + multiple - 1) / multiple * multiple;
      ext[i] = padded;
    }
  }
  if (padded < 0) tir::throw_error("DescMismatch", "block '" + block + "' has no channel reduction 'vrc'");
  s.cache_read(block, 0, "global");
  s.cache_read(block, 1, "global");
  s.pad_block(block, ext);
  widen_reads(s, block);
  return padded;
}

void register_tensorize_step_handler() {
  static const bool registered = [] {
    tir::register_step_handler("b200.tensorize", [](tir::Schedule& s, const tir::TraceStep& step) {
      replace_with_call(s, step.args.at("block").get<std::string>(), step.args.at("intrin").get<std::string>(),
                        step.args.value("drop_init", false));
    });
    return true;
  }();
  (void)registered;
}

}  // namespace tir_b200
