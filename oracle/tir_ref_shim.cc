// tir_ref_shim.cc — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A minimal extern "C" surface over the reference interpreter so Python tests
// (golden vectors) and bench.py's CPU-baseline leg can run tir::run
// (/root/reference/proj/src/interp.cc:579-590) on programs written in the
// reference grammar (parse_text, src/parser.cc:801). Built by oracle/Makefile
// against the unmodified reference sources into oracle/_ref/.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tir/interp.h"
#include "tir/text.h"
#include "testing/workloads.h"

namespace {
thread_local std::string g_err;

int fail(const std::string& msg) {
  g_err = msg;
  return -1;
}

// Runs one program. inputs[i] holds input param i (input_params order,
// interp.cc:189-197) as f32 storage (F16 is an f32 tag, ir.cc:36-47).
int run_one(const char* ir_text, int n_in, const float* const* inputs, float* out,
            int64_t out_elems, double* wall, int64_t* intrinsic_calls) {
  try {
    tir::PrimFuncPtr f = tir::parse_text(ir_text);
    auto in_params = tir::input_params(*f);
    if (static_cast<int>(in_params.size()) != n_in) {
      return fail("program expects " + std::to_string(in_params.size()) + " inputs, got " +
                  std::to_string(n_in));
    }
    std::vector<tir::TensorValue> values;
    for (int i = 0; i < n_in; ++i) {
      tir::TensorValue t = tir::TensorValue::zeros(in_params[i]->dtype, in_params[i]->shape);
      if (!tir::dtype_is_float(t.dtype)) return fail("shim supports float inputs only");
      std::memcpy(t.data.data(), inputs[i], t.data.size());
      values.push_back(std::move(t));
    }
    tir::ExecContext ctx;
    auto t0 = std::chrono::steady_clock::now();
    auto outs = tir::run(*f, values, ctx);
    auto t1 = std::chrono::steady_clock::now();
    if (wall) *wall = std::chrono::duration<double>(t1 - t0).count();
    if (intrinsic_calls) *intrinsic_calls = ctx.counters.intrinsic_calls;
    if (out) {
      if (outs.empty()) return fail("program has no output");
      const tir::TensorValue& o = outs[0];
      if (o.num_elements() != out_elems) {
        return fail("output has " + std::to_string(o.num_elements()) + " elements, caller gave " +
                    std::to_string(out_elems));
      }
      std::memcpy(out, o.data.data(), static_cast<size_t>(out_elems) * 4);
    }
    return 0;
  } catch (const tir::Error& e) {
    return fail(e.kind() + ": " + e.message());
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}
}  // namespace

extern "C" {

const char* tirref_last_error(void) { return g_err.c_str(); }

int tirref_run(const char* ir_text, int n_in, const float* const* inputs, float* out,
               int64_t out_elems, double* wall_seconds, int64_t* intrinsic_calls) {
  return run_one(ir_text, n_in, inputs, out, out_elems, wall_seconds, intrinsic_calls);
}

// Runs `n_prog` independent programs concurrently, one std::thread each, each
// with its own parsed PrimFunc and ExecContext (the reference is re-entrant
// across contexts). inputs[p*n_in + i] is input i of program p;
// outs[p] (may be null) receives program p's first output. Returns the
// wall-clock seconds of the whole batch in *wall_seconds.
int tirref_run_many(int n_prog, const char* const* ir_texts, int n_in, const float* const* inputs,
                    float* const* outs, const int64_t* out_elems, double* wall_seconds) {
  std::vector<int> rc(n_prog, 0);
  std::vector<std::string> errs(n_prog);
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> threads;
  for (int p = 0; p < n_prog; ++p) {
    threads.emplace_back([&, p] {
      rc[p] = run_one(ir_texts[p], n_in, inputs + static_cast<size_t>(p) * n_in,
                      outs ? outs[p] : nullptr, out_elems ? out_elems[p] : 0, nullptr, nullptr);
      if (rc[p]) errs[p] = g_err;
    });
  }
  for (auto& t : threads) t.join();
  auto t1 = std::chrono::steady_clock::now();
  if (wall_seconds) *wall_seconds = std::chrono::duration<double>(t1 - t0).count();
  for (int p = 0; p < n_prog; ++p) {
    if (rc[p]) return fail("program " + std::to_string(p) + ": " + errs[p]);
  }
  return 0;
}

// The reference's own seeded input generator, random_tensor
// (proj/tests/testing/workloads.h:170-184), for `count` f32 elements.
int tirref_random_tensor(int64_t count, uint64_t seed, float* out) {
  try {
    tir::TensorValue t = tir::testing::random_tensor(tir::DType::F32, {count}, seed);
    std::memcpy(out, t.data.data(), static_cast<size_t>(count) * 4);
    return 0;
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}

// The reference's own workload sources (workloads.h:35-166), so tests can run
// exactly the programs the reference tests run. which: "matmul" (a=n),
// "gemm_relu" (a=n), "conv2d" (h,w,ci,kh,kw,co), "depthwise" (h,w,c,kh,kw).
const char* tirref_workload_source(const char* which, int a, int b, int c, int d, int e, int f) {
  static thread_local std::string src;
  std::string w(which);
  if (w == "matmul") {
    src = tir::testing::matmul_source(a);
  } else if (w == "gemm_relu") {
    src = tir::testing::gemm_relu_source(a);
  } else if (w == "conv2d") {
    src = tir::testing::conv2d_source(a, b, c, d, e, f);
  } else if (w == "depthwise") {
    src = tir::testing::depthwise_source(a, b, c, d, e);
  } else {
    fail("unknown workload '" + w + "'");
    return nullptr;
  }
  return src.c_str();
}

// The reference's tensor-file I/O (interp.cc:730-769), so golden vectors on
// disk are written and read by the reference itself. dtype: "f32" / "f16" (f16
// is stored as f32 bits, ir.cc:36-47).
int tirref_write_tensor(const char* path, const char* dtype, int ndim, const int64_t* shape,
                        const float* data) {
  try {
    std::string d(dtype);
    tir::DType dt = d == "f16" ? tir::DType::F16 : tir::DType::F32;
    tir::TensorValue t = tir::TensorValue::zeros(dt, std::vector<int64_t>(shape, shape + ndim));
    std::memcpy(t.data.data(), data, t.data.size());
    tir::write_tensor(path, t);
    return 0;
  } catch (const tir::Error& e) {
    return fail(e.kind() + ": " + e.message());
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}

// Reads a tensor file; returns the element count (or -1), the shape in
// shape_out[0..*ndim) (at most 8 dims) and up to `cap` elements as f32.
int64_t tirref_read_tensor(const char* path, float* out, int64_t cap, int64_t* shape_out, int* ndim) {
  try {
    tir::TensorValue t = tir::read_tensor(path);
    if (!tir::dtype_is_float(t.dtype)) return fail("float tensors only");
    *ndim = static_cast<int>(t.shape.size());
    for (size_t i = 0; i < t.shape.size() && i < 8; ++i) shape_out[i] = t.shape[i];
    const int64_t n = t.num_elements();
    if (out) std::memcpy(out, t.data.data(), static_cast<size_t>(std::min(n, cap)) * 4);
    return n;
  } catch (const tir::Error& e) {
    return fail(e.kind() + ": " + e.message());
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}

// tir::run over inputs read from tensor files, first output written to a
// tensor file: a golden vector produced end to end by the reference.
int tirref_run_files(const char* ir_text, int n_in, const char* const* in_paths, const char* out_path) {
  try {
    tir::PrimFuncPtr f = tir::parse_text(ir_text);
    std::vector<tir::TensorValue> values;
    for (int i = 0; i < n_in; ++i) values.push_back(tir::read_tensor(in_paths[i]));
    tir::ExecContext ctx;
    auto outs = tir::run(*f, values, ctx);
    if (outs.empty()) return fail("program has no output");
    tir::write_tensor(out_path, outs[0]);
    return 0;
  } catch (const tir::Error& e) {
    return fail(e.kind() + ": " + e.message());
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}

}  // extern "C"
