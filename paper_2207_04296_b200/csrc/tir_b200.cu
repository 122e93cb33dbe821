// tir_b200.cu — the C-ABI (include/tir_b200.h): operator planning, TMA
// descriptor encoding, kernel launches, host-buffer entry points.
//
// Each entry point replaces the body of one reference HostKernel
// (/root/reference/proj/include/tir/interp.h:120): the adapter
// (paper_2207_04296_b200/adapter/) turns the views of a tensorized block
// (src/interp.cc:371-373) into one of these calls.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tir_b200.h"
#include "dep.cuh"
#include "halo.cuh"
#include "igemm.cuh"
#include "netops.cuh"
#include "options.h"
#include "prep.cuh"
#include "rowpack.cuh"

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;
thread_local unsigned long long* g_trace = nullptr;

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return set_err(TIR_B200_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                                \
  } while (0)

// ------------------------------------------------------------------ driver API

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Driver {
  EncodeTiledFn tiled = nullptr;   // the caching wrappers below
  EncodeIm2colFn im2col = nullptr;
  int version = 0;
};

EncodeTiledFn g_encode_tiled = nullptr;   // the driver's entry points
EncodeIm2colFn g_encode_im2col = nullptr;

// Tensor-map encodes are a few microseconds of host time each and a call plans
// 2-3 of them; repeated calls on the same buffers (graph capture loops, the
// host-buffer pipeline's per-chunk launches) re-encode identical maps. A small
// per-thread cache keyed by every encode argument returns the previous result.
struct EncodeKey {
  uint64_t w[40];
  int n = 0;
  void put(uint64_t v) { w[n++] = v; }
  bool operator==(const EncodeKey& o) const { return n == o.n && std::memcmp(w, o.w, n * sizeof(uint64_t)) == 0; }
};
struct EncodeCache {
  static constexpr int kSize = 32;
  EncodeKey key[kSize];
  CUtensorMap map[kSize];
  int next = 0;
  bool find(const EncodeKey& k, CUtensorMap* out) const {
    for (int i = 0; i < kSize; ++i)
      if (key[i] == k) {
        *out = map[i];
        return true;
      }
    return false;
  }
  void put(const EncodeKey& k, const CUtensorMap& m) {
    key[next] = k;
    map[next] = m;
    next = (next + 1) % kSize;
  }
};
thread_local EncodeCache t_encode_cache;

CUresult encode_tiled_cached(CUtensorMap* m, CUtensorMapDataType dt, cuuint32_t rank, void* ptr,
                             const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                             const cuuint32_t* es, CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                             CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob) {
  EncodeKey k;
  k.put(1);
  k.put(dt);
  k.put(rank);
  k.put(reinterpret_cast<uintptr_t>(ptr));
  for (cuuint32_t i = 0; i < rank; ++i) k.put(dims[i]);
  for (cuuint32_t i = 0; i + 1 < rank; ++i) k.put(strides[i]);
  for (cuuint32_t i = 0; i < rank; ++i) k.put((static_cast<uint64_t>(box[i]) << 32) | es[i]);
  k.put((static_cast<uint64_t>(il) << 48) | (static_cast<uint64_t>(sw) << 32) | (static_cast<uint64_t>(l2) << 16) | oob);
  if (t_encode_cache.find(k, m)) return CUDA_SUCCESS;
  const CUresult r = g_encode_tiled(m, dt, rank, ptr, dims, strides, box, es, il, sw, l2, oob);
  if (r == CUDA_SUCCESS) t_encode_cache.put(k, *m);
  return r;
}

CUresult encode_im2col_cached(CUtensorMap* m, CUtensorMapDataType dt, cuuint32_t rank, void* ptr,
                              const cuuint64_t* dims, const cuuint64_t* strides, const int* lo, const int* hi,
                              cuuint32_t ch, cuuint32_t px, const cuuint32_t* es, CUtensorMapInterleave il,
                              CUtensorMapSwizzle sw, CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob) {
  EncodeKey k;
  k.put(2);
  k.put(dt);
  k.put(rank);
  k.put(reinterpret_cast<uintptr_t>(ptr));
  for (cuuint32_t i = 0; i < rank; ++i) k.put(dims[i]);
  for (cuuint32_t i = 0; i + 1 < rank; ++i) k.put(strides[i]);
  for (cuuint32_t i = 0; i + 2 < rank; ++i)
    k.put((static_cast<uint64_t>(static_cast<uint32_t>(lo[i])) << 32) | static_cast<uint32_t>(hi[i]));
  k.put((static_cast<uint64_t>(ch) << 32) | px);
  for (cuuint32_t i = 0; i < rank; ++i) k.put(es[i]);
  k.put((static_cast<uint64_t>(il) << 48) | (static_cast<uint64_t>(sw) << 32) | (static_cast<uint64_t>(l2) << 16) | oob);
  if (t_encode_cache.find(k, m)) return CUDA_SUCCESS;
  const CUresult r = g_encode_im2col(m, dt, rank, ptr, dims, strides, lo, hi, ch, px, es, il, sw, l2, oob);
  if (r == CUDA_SUCCESS) t_encode_cache.put(k, *m);
  return r;
}

const Driver* driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess) {
      g_encode_tiled = reinterpret_cast<EncodeTiledFn>(fn);
      d.tiled = encode_tiled_cached;
    }
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess) {
      g_encode_im2col = reinterpret_cast<EncodeIm2colFn>(fn);
      d.im2col = encode_im2col_cached;
    }
    cudaDriverGetVersion(&d.version);
  });
  return &d;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size: a
// driver call per launch otherwise (host-side planning cost of every call).
cudaError_t ensure_smem_ptr(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, size_t>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const void* key = reinterpret_cast<const char*>(func) + dev;  // per device
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : done)
      if (e.first == key && e.second >= bytes) return cudaSuccess;
  }
  const cudaError_t r = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (r == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : done)
      if (e.first == key) {
        e.second = std::max(e.second, bytes);
        return r;
      }
    done.emplace_back(key, bytes);
  }
  return r;
}

template <typename Params>
cudaError_t ensure_smem(void (*kernel)(Params), size_t bytes) {
  return ensure_smem_ptr(reinterpret_cast<const void*>(kernel), bytes);
}

struct DeviceInfo {
  int sms = 148;
  int smem_optin = 227 * 1024;
};

DeviceInfo device_info() {
  static std::mutex mu;
  static DeviceInfo cache[64];
  static bool have[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && !have[dev]) {
    cudaDeviceGetAttribute(&cache[dev].sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&cache[dev].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    have[dev] = true;
  }
  return cache[(dev >= 0 && dev < 64) ? dev : 0];
}

CUtensorMapSwizzle swizzle_for(int row_bytes) {
  switch (row_bytes) {
    case 128: return CU_TENSOR_MAP_SWIZZLE_128B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    default: return CU_TENSOR_MAP_SWIZZLE_NONE;
  }
}

// Row-major [rows, cols] fp16 matrix, box {box_cols, box_rows}.
int encode_2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int box_cols,
              int box_rows) {
  const Driver* d = driver();
  if (!d->tiled) return set_err(TIR_B200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = d->tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle_for(box_cols * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(TIR_B200_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld box=%dx%d",
                   static_cast<int>(r), static_cast<long long>(rows), static_cast<long long>(cols),
                   box_cols, box_rows);
  return TIR_B200_OK;
}

// ------------------------------------------------------------------ geometry

struct Geo {
  int64_t n, in[3], ci, co, k[3], s[3], p[3], d[3], g, out[3];  // [0]=D,[1]=H,[2]=W
  bool transposed;
};

int make_geo(const tir_b200_conv_desc* desc, Geo* g) {
  if (!desc) return set_err(TIR_B200_ERR_VALUE, "null descriptor");
  g->n = desc->n;
  g->in[0] = desc->in_d; g->in[1] = desc->in_h; g->in[2] = desc->in_w;
  g->ci = desc->ci; g->co = desc->co;
  g->k[0] = desc->k_d; g->k[1] = desc->k_h; g->k[2] = desc->k_w;
  g->s[0] = desc->s_d; g->s[1] = desc->s_h; g->s[2] = desc->s_w;
  g->p[0] = desc->p_d; g->p[1] = desc->p_h; g->p[2] = desc->p_w;
  g->d[0] = desc->d_d; g->d[1] = desc->d_h; g->d[2] = desc->d_w;
  g->g = desc->groups;
  g->transposed = desc->transposed != 0;
  if (g->n < 1 || g->ci < 1 || g->co < 1 || g->g < 1)
    return set_err(TIR_B200_ERR_VALUE, "conv: n, ci, co, groups must be >= 1");
  if (g->ci % g->g || g->co % g->g)
    return set_err(TIR_B200_ERR_VALUE, "conv: groups must divide ci and co");
  for (int i = 0; i < 3; ++i) {
    if (g->in[i] < 1 || g->k[i] < 1 || g->s[i] < 1 || g->p[i] < 0 || g->d[i] < 1)
      return set_err(TIR_B200_ERR_VALUE, "conv: bad extents/stride/padding/dilation");
    if (g->transposed) {
      g->out[i] = (g->in[i] - 1) * g->s[i] - 2 * g->p[i] + g->d[i] * (g->k[i] - 1) + 1;
    } else {
      int64_t span = g->in[i] + 2 * g->p[i] - g->d[i] * (g->k[i] - 1) - 1;
      if (span < 0) return set_err(TIR_B200_ERR_VALUE, "conv: kernel larger than padded input");
      g->out[i] = span / g->s[i] + 1;
    }
    if (g->out[i] < 1) return set_err(TIR_B200_ERR_VALUE, "conv: empty output");
  }
  const int64_t in_elems = g->n * g->in[0] * g->in[1] * g->in[2] * g->ci;
  const int64_t out_elems = g->n * g->out[0] * g->out[1] * g->out[2] * g->co;
  if (in_elems >= (1ll << 31) * 8 || out_elems >= (1ll << 31) * 8)
    return set_err(TIR_B200_ERR_UNSUPPORTED, "conv: tensor too large");
  return TIR_B200_OK;
}

bool is_depthwise(const Geo& g) { return g.g == g.ci && g.ci == g.co && !g.transposed; }

// ------------------------------------------------------------------ workspace

// Relayout scratch (channel pad, (kw, c) / (kh, kw, c) packing), one buffer per
// (device, stream): kernels on one stream are ordered, so calls that share a
// stream may share its buffer; two streams never do. Grow-only and never freed
// while the process runs: a CUDA graph captured over a relayout keeps the raw
// pointer, so a later, larger request gets a NEW buffer and the old one stays
// valid (retired, not freed). tir_b200_release_workspaces() frees everything
// once the caller knows no graph or in-flight launch references it.
struct Workspace {
  int dev = -1;
  cudaStream_t stream = nullptr;
  void* ptr = nullptr;
  size_t bytes = 0;
};
std::mutex g_ws_mu;
std::vector<Workspace> g_ws;       // live buffers, one per (device, stream)
std::vector<void*> g_ws_retired;   // outgrown buffers (may still be referenced by graphs)

int workspace(size_t bytes, cudaStream_t stream, void** out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  for (Workspace& w : g_ws) {
    if (w.dev != dev || w.stream != stream) continue;
    if (w.bytes < bytes) {
      void* p = nullptr;
      CUDA_TRY(cudaMalloc(&p, bytes));
      g_ws_retired.push_back(w.ptr);
      w.ptr = p;
      w.bytes = bytes;
    }
    *out = w.ptr;
    return TIR_B200_OK;
  }
  Workspace w;
  w.dev = dev;
  w.stream = stream;
  w.bytes = bytes;
  CUDA_TRY(cudaMalloc(&w.ptr, bytes));
  g_ws.push_back(w);
  *out = w.ptr;
  return TIR_B200_OK;
}

// ------------------------------------------------------------------ launches

// Programmatic dependent launch: the kernel may begin (prologue, TMEM alloc,
// barrier init) while the previous kernel on the stream drains; it waits with
// griddepcontrol.wait before touching global memory. Captured into CUDA graphs
// as a programmatic edge. TIR_B200_NO_PDL=1 disables it.
template <typename Params>
cudaError_t launch_pdl(void (*kernel)(Params), int grid, int block, size_t smem, cudaStream_t stream,
                       const Params& p) {
  const bool no_pdl = tb::options().no_pdl != 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, p);
}

// Same, as clusters of `cluster` CTAs along x (CTA pairs for cta_group::2 kernels).
template <typename Params>
cudaError_t launch_pdl_cluster(void (*kernel)(Params), int grid, int cluster, int block, size_t smem,
                               cudaStream_t stream, const Params& p) {
  const bool no_pdl = tb::options().no_pdl != 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, p);
}

// ------------------------------------------------------------------ igemm launch

// CTA pairs for plain GEMMs: tiled A, streamed row-major B in >= 2 chunks, one
// problem (no groups / split-K / batch / sub-problems), an even M-tile count:
// tcgen05.mma.cta_group::2 (p.mc = 2; each SM loads and reads half of B).
// Measured on B200, vs unpaired: 8192^3 1094 -> 1290 TFLOPS, BERT-large QKV /
// FFN1 / FFN2 GEMMs -11 / -12 / -15 %. (A B-multicast-only pair was measured
// too: +4-7 % at 8192^3, nothing below; removed.) TIR_B200_MC=0 disables pairs.
constexpr int kNotEligible = -100;  // a specialised path declines; the caller takes the general one

bool use_pairs(const tb::IgemmParams& p, int bn) {
  if (!tb::options().mc) return false;
  return p.a_mode == tb::A_TILED && p.b_mode == tb::B_STREAM && !p.b_kmajor && p.num_sub == 1 &&
         p.groups == 1 && p.ksplit == 1 && !p.batch_tiles && bn >= 128 && p.sub[0].tiles_m % 2 == 0 &&
         p.total_tiles == p.sub[0].tiles_m * p.tiles_n;
}

template <int BN, int KS, bool EPI8, bool GP = false>
int launch_igemm_bn(tb::IgemmParams& p, cudaStream_t stream) {
  using Cfg = tb::IgemmCfg<BN, KS, EPI8, GP>;
  const DeviceInfo di = device_info();
  p.l2_prefetch = tb::options().igemm_prefetch;
  const int table = p.total_pieces * 16;
  // Stage the bias in shared memory for the TMA-store epilogue when it is small
  // and every 32-column chunk starts 16-byte aligned inside it.
  // Only for short-K (epilogue-bound) tiles: K-heavy GEMMs need the shared memory for pipeline stages.
  int nst_all = 0;
  for (int i = 0; i < p.num_sub; ++i) nst_all = std::max(nst_all, p.sub[i].num_stages);
  const int nbias = p.groups * p.cog;
  p.bias_floats = (p.bias && p.store_mode && !p.batch_tiles && nst_all * KS * tb::kBK <= 256 && nbias <= 4096 &&
                   p.cog % 32 == 0 &&
                   (reinterpret_cast<uintptr_t>(p.bias) & 15) == 0 && !tb::options().no_smem_bias)
                      ? (nbias + 3) / 4 * 4 : 0;
  // the staged bias must not cost the ring its second stage
  if (p.bias_floats && di.smem_optin - 1280 - table - p.bias_floats * 4 - Cfg::kEpiBytes <
                           2 * (Cfg::kABytes + Cfg::kBBytes))
    p.bias_floats = 0;
  const int budget = di.smem_optin - 1024 - 256 - table - p.bias_floats * 4 - Cfg::kEpiBytes;
  int nst_max = 0;
  for (int i = 0; i < p.num_sub; ++i) nst_max = std::max(nst_max, p.sub[i].num_stages);
  const int keys = p.groups * p.tiles_n * p.ksplit;  // CTAs per B-panel cycle
  // GP: the panel is the packed groups' own [taps*cig, 32] blocks (not stage-padded)
  const int res_rows = GP ? p.gp_taps * p.gp_kpg * 16 : nst_max * Cfg::kBRows;
  const int res_bytes = res_rows * BN * 2;
  int grid = std::min(p.total_tiles, di.sms);
  // Keep B resident when its whole K panel fits next to a >= 3-deep A ring and
  // every CTA can be pinned to one (group, n-tile): grid a multiple of `keys`.
  if (p.b_mode == tb::B_STREAM && p.num_sub == 1 && !p.batch_tiles && p.ksplit == 1 && keys <= di.sms &&
      res_rows * Cfg::kBRowBytes < (1 << 18) && res_bytes + 3 * Cfg::kABytes <= budget) {
    p.b_mode = tb::B_RESIDENT;
    p.b_res_rows = res_rows;
    p.stages = std::min(8, (budget - res_bytes) / Cfg::kABytes);
    grid = std::min(p.total_tiles, di.sms / keys * keys);
  } else {
    if (GP) return kNotEligible;  // GP reads its panel resident only
    p.b_res_rows = 0;
    p.stages = std::min(8, budget / (Cfg::kABytes + Cfg::kBBytes));
  }
  if (p.stages < 2) return set_err(TIR_B200_ERR_UNSUPPORTED, "not enough shared memory");
  size_t smem = Cfg::smem_bytes(p.stages, p.b_res_rows, p.total_pieces, p.bias_floats);
  if (p.ksplit > 1) {
    // one output tile per CTA, its ksplit partials in one cluster; the [128][BN + 4]
    // fp32 partial image reuses the drained operand ring
    const size_t ring = static_cast<size_t>(p.stages) * Cfg::kABytes +
                        (p.b_res_rows ? static_cast<size_t>(p.b_res_rows) * BN * 2
                                      : static_cast<size_t>(p.stages) * Cfg::kBBytes);
    if (p.total_tiles > di.sms || p.total_tiles % p.ksplit || ring < static_cast<size_t>(tb::kBM) * (BN + 4) * 4)
      return set_err(TIR_B200_ERR_UNSUPPORTED, "split-K plan does not fit (tiles %d, ksplit %d)", p.total_tiles,
                     p.ksplit);
    CUDA_TRY(ensure_smem(tb::igemm_tc_kernel<BN, KS, EPI8>, smem));
    p.mc = 0;
    p.trace = g_trace;
    CUDA_TRY(launch_pdl_cluster(tb::igemm_tc_kernel<BN, KS, EPI8>, p.total_tiles, p.ksplit, Cfg::kThreadsN, smem,
                                stream, p));
    ++g_launches;
    return TIR_B200_OK;
  }
  if constexpr (GP) {
    if (p.ksplit != 1) return kNotEligible;
    CUDA_TRY(ensure_smem(tb::igemm_tc_kernel<BN, KS, EPI8, false, true>, smem));
    if (const int e = tb::options().max_ctas) grid = std::max(1, std::min(grid, e));
    p.mc = 0;
    p.trace = g_trace;
    CUDA_TRY(launch_pdl(tb::igemm_tc_kernel<BN, KS, EPI8, false, true>, grid, Cfg::kThreadsN, smem, stream, p));
    ++g_launches;
    return TIR_B200_OK;
  } else {
  CUDA_TRY(ensure_smem(tb::igemm_tc_kernel<BN, KS, EPI8>, smem));
  // B-multicast CTA pairs (igemm.cuh mc_tile) for plain GEMMs with wide N tiles.
  p.mc = 0;
  if (use_pairs(p, BN) && grid >= 2) {
    static int max_clusters = -1;  // per instantiation: same smem / block for every launch that gets here
    if (max_clusters < 0) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(di.sms / 2 * 2);
      cfg.blockDim = dim3(Cfg::kThreadsN);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      max_clusters = cudaOccupancyMaxActiveClusters(&n, tb::igemm_tc_kernel<BN, KS, EPI8>, &cfg) == cudaSuccess
                         ? n : 0;
      cudaGetLastError();
    }
    if (max_clusters > 0 && BN >= 128) {
      p.mc = 2;  // tcgen05.mma.cta_group::2 (M = 256, B split by column)
      grid = std::min(grid / 2, max_clusters) * 2;
    }
  }
  if (p.mc == 2) {  // half of B per slot: a deeper ring in the same shared memory
    p.stages = std::min(8, budget / (Cfg::kABytes + Cfg::kBBytes / 2));
    smem = Cfg::smem_bytes(p.stages, 0, p.total_pieces, p.bias_floats, true);
  }
  if (const int e = tb::options().max_ctas)
    grid = p.mc ? std::max(2, std::min(grid, e / 2 * 2)) : std::max(1, std::min(grid, e));
  p.trace = g_trace;
  if (p.mc == 2) {
    if constexpr (BN >= 128) {
      CUDA_TRY(ensure_smem(tb::igemm_tc_kernel<BN, KS, EPI8, true>, smem));
      CUDA_TRY(launch_pdl_cluster(tb::igemm_tc_kernel<BN, KS, EPI8, true>, grid, 2, Cfg::kThreadsN, smem, stream,
                                  p));
    }
  } else {
    CUDA_TRY(launch_pdl(tb::igemm_tc_kernel<BN, KS, EPI8>, grid, Cfg::kThreadsN, smem, stream, p));
  }
  ++g_launches;
  return TIR_B200_OK;
  }  // !GP
}

// Short-K tiles (<= 1024-deep reduction, no split-K) with a wide, fused fp16 /
// bias / activation epilogue — the networks' 1x1 convs, expansion GEMMs and
// attention — are epilogue-bound: they take the 8-epilogue-warp variant
// (IgemmCfg EPI8). Measured: ResNet-50 forward -8%, MobileNet-V2 -13%; the
// paper's fp32-output convs keep 4 producers (GRP / DIL lose 5-8% with 3).
bool use_epi8(const tb::IgemmParams& p, int bn, int ks) {
  if (tb::options().epi8 >= 0) return tb::options().epi8 != 0;
  int nst = 0;
  for (int i = 0; i < p.num_sub; ++i) nst = std::max(nst, p.sub[i].num_stages);
  const bool fused = p.out_f16 || p.bias || p.relu || p.residual;
  // up to K = 1024 per tile (measured on BERT-large: QKV / out / FFN1 GEMMs -5 / -5 / -22 %,
  // FFN2 with K = 4096 +3 %)
  // narrow im2col pieces (< 64 channels) are TMA-request-bound: keep 4 producers
  // a 64-column tile with K >= 512 is load-bound, not epilogue-bound: keep 4 producers
  // (BERT attention P.V: 13.6 -> 12.3 us)
  if (bn == 64 && nst * ks * tb::kBK >= 512) return false;
  return p.ksplit <= 1 && nst * ks * tb::kBK <= 1024 && bn >= 64 && fused && p.a_box_ch == 64;
}

template <int BN>
int launch_igemm_ks(tb::IgemmParams& p, int ks, cudaStream_t stream) {
  const bool e8 = use_epi8(p, BN, ks);
  switch (ks) {
    case 4: return e8 ? launch_igemm_bn<BN, 4, true>(p, stream) : launch_igemm_bn<BN, 4, false>(p, stream);
    case 2: return e8 ? launch_igemm_bn<BN, 2, true>(p, stream) : launch_igemm_bn<BN, 2, false>(p, stream);
    default: return e8 ? launch_igemm_bn<BN, 1, true>(p, stream) : launch_igemm_bn<BN, 1, false>(p, stream);
  }
}

int launch_igemm_gp(tb::IgemmParams& p, int bn, int ks, cudaStream_t stream) {
  if (bn == 128) return ks >= 2 ? launch_igemm_bn<128, 2, false, true>(p, stream)
                                : launch_igemm_bn<128, 1, false, true>(p, stream);
  if (bn == 64) return ks >= 2 ? launch_igemm_bn<64, 2, false, true>(p, stream)
                               : launch_igemm_bn<64, 1, false, true>(p, stream);
  return kNotEligible;
}

int launch_igemm(tb::IgemmParams& p, int bn, int ks, cudaStream_t stream) {
  switch (bn) {
    case 16: return launch_igemm_ks<16>(p, ks, stream);
    case 32: return launch_igemm_ks<32>(p, ks, stream);
    case 64: return launch_igemm_ks<64>(p, ks, stream);
    case 128: return launch_igemm_ks<128>(p, std::min(ks, 2), stream);
    case 256: return launch_igemm_ks<256>(p, std::min(ks, 2), stream);
  }
  return set_err(TIR_B200_ERR_UNSUPPORTED, "no kernel for BN=%d", bn);
}

// K sub-blocks (64 deep) per pipeline stage: the largest of {4, 2, 1} whose
// padding waste (pieces past the end of the reduction) is minimal, capped by
// shared memory (two stages of A + B must fit). Narrow-piece convs (box < 64
// channels: the packed CI = 3 stems) never take the 8-warp epilogue, so their
// two stages may use everything but the 4-warp staging (DIL: one 256-deep stage
// per tile instead of two, 36.9 -> 34.9 us).
int choose_ks(int max_pieces, int box, int bn) {
  if (const int e = tb::options().ks) return std::max(1, std::min(4, e));
  const int pps1 = tb::kBK / box;
  const int limit = (box < 64 && !tb::options().ks_strict) ? 227 * 1024 - 1280 - 4 * 8192 - 16 * max_pieces - 512
                                                                 : 190 * 1024;
  int best = 1;
  int64_t best_waste = -1;
  for (int ks : {4, 2, 1}) {
    if (2 * ks * (16384 + 64 * bn * 2) > limit) continue;  // two stages must fit
    const int64_t per = static_cast<int64_t>(pps1) * ks;
    const int64_t waste = (max_pieces + per - 1) / per * per - max_pieces;
    if (waste * 8 <= max_pieces) return ks;  // <= 12.5% padded MMA work: deepest such stage
    if (best_waste < 0 || waste < best_waste) {
      best = ks;
      best_waste = waste;
    }
  }
  return best;
}

// Y as a 2-D [rows, ldy] map for the per-warp TMA-store epilogue.
// Box {cw, 32}: one epilogue warp's 32 rows x a staged chunk of cw columns
// (32; 64 for fp16 output when BN >= 64 and no chunk crosses a group, so every
// staged row is 128 bytes), swizzled like the staging buffer.
int encode_y(tb::IgemmParams& p, void* Y, int64_t rows, int out_f16, int bn) {
  const Driver* d = driver();
  if (!d->tiled) return set_err(TIR_B200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int esz = out_f16 ? 2 : 4;
  p.epi_cw = (out_f16 && bn >= 64 && (p.groups == 1 || p.cog % 64 == 0)) ? 64 : 32;
  const int row_bytes = p.epi_cw * esz;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.ldy), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.ldy) * esz};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(p.epi_cw), 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = d->tiled(&p.tmY, out_f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                        Y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(TIR_B200_ERR_CUDA, "Y tensor map failed (%d)", (int)r);
  return TIR_B200_OK;
}

// Fused epilogue (bias + ReLU) resolved from the C-ABI's optional struct.
struct Epi {
  const float* bias = nullptr;
  int relu = 0;
  const uint16_t* residual = nullptr;
  bool on() const { return bias != nullptr || relu != 0 || residual != nullptr; }
  void apply(tb::IgemmParams& p) const { p.bias = bias; p.relu = relu; p.residual = residual; }
};

Epi make_epi(const tir_b200_epilogue* e) {
  Epi r;
  if (e) {
    r.bias = e->bias;
    r.relu = e->relu;
    r.residual = e->residual;
  }
  return r;
}

// Store mode for row-linear outputs: TMA store when every 32-column chunk lies
// inside one group (or there is a single group), reduce-add for in-place
// accumulate; otherwise the generic per-row path.
int pick_store_mode(tb::IgemmParams& p, int bn, void* Y, const float* Yin, int64_t rows, int accumulate,
                    int out_f16) {
  p.store_mode = 0;
  if (tb::options().no_tma_store) return TIR_B200_OK;
  // Reduce-add cannot apply the epilogue after the add (the ABI order is
  // (Yin + acc) + bias + residual, then the activation): accumulate + epilogue stays generic.
  if (accumulate && (p.bias || p.relu || p.residual)) return TIR_B200_OK;
  if (bn < 32 || !(p.groups == 1 || p.cog % 32 == 0) || (accumulate && Yin != Y)) return TIR_B200_OK;
  if ((reinterpret_cast<uintptr_t>(Y) & 15) || (p.ldy * (out_f16 ? 2 : 4)) % 16) return TIR_B200_OK;
  int rc = encode_y(p, Y, rows, out_f16, bn);
  if (rc) return rc;
  p.store_mode = accumulate ? 2 : 1;
  return TIR_B200_OK;
}

// Chooses the N tile by a tensor-issue cost model measured on B200
// (tools/mma_rate.cu): one M=128, K=16 MMA takes max(N/2, 32 + N/4) cycles
// (SMEM operand bandwidth caps small N). Time ~ waves x k_steps x cycles/MMA,
// with waves = ceil(tiles / SMs). A narrower tile must be >= 20% cheaper to
// win: the model ignores the extra L2 traffic of re-reading A per N tile.
int choose_bn(int64_t cols, int64_t m_tiles, int64_t groups, int64_t k_steps, int sms, bool plain_f32 = false) {
  if (const int e = tb::options().bn) return e;
  int bn_max = 16;
  while (bn_max < cols && bn_max < 256) bn_max *= 2;
  int best = bn_max;
  double best_cost = -1;
  // N = 16 only for 16-column outputs: below 32 columns the TMA-store epilogue
  // is unavailable and the generic one costs more than the model's MMA saving
  // (measured: C1D 5.8 -> 4.9 us at N = 32).
  const int bn_min = cols <= 16 ? 16 : 32;
  for (int bn = bn_max; bn >= bn_min; bn /= 2) {
    const int64_t tiles = m_tiles * groups * ((cols + bn - 1) / bn);
    const int64_t waves = (tiles + sms - 1) / sms;
    const double cyc = std::max(bn / 2.0, 32.0 + bn / 4.0);
    // Plain fp32-output launches (the paper's ops) add the last tile's epilogue, which
    // nothing overlaps: 128 x bn fp32 through TMEM -> staging -> TMA store at ~64 B/clk
    // (measured: C1D 4.76 -> 4.47 us at N = 32). Fused fp16 network layers keep the
    // MMA-only model (with the term MobileNet-V2 lost 4 %).
    const double cost = static_cast<double>(waves) * static_cast<double>(k_steps) * cyc +
                        (plain_f32 ? 128.0 * bn * 4 / 64 : 0.0);
    if (best_cost < 0 || cost < best_cost * 0.8) {
      best = bn;
      best_cost = cost;
    }
  }
  return best;
}

void set_sub_identity(tb::SubProb& s) {
  for (int i = 0; i < 3; ++i) {
    s.a_lo[i] = 0; s.a_st[i] = 1; s.taps[i] = 1; s.a_dil[i] = 1;
    s.w_base[i] = 0; s.w_step[i] = 1; s.o_st[i] = 1; s.o_b[i] = 0;
  }
}

int finalize_tiles(tb::IgemmParams& p, int bn, int ks) {
  p.tiles_n = static_cast<int32_t>((p.cog + bn - 1) / bn);
  int64_t t = 0, pieces = 0;
  for (int i = 0; i < p.num_sub; ++i) {
    tb::SubProb& s = p.sub[i];
    s.piece_begin = static_cast<int32_t>(pieces);
    if (p.a_mode != tb::A_TILED) pieces += s.num_pieces;
    s.tiles_m = (s.m_count + tb::kBM - 1) / tb::kBM;
    s.tile_begin = static_cast<int32_t>(t);
    t += static_cast<int64_t>(s.tiles_m) * p.groups * p.tiles_n * p.ksplit;
    const int pps = ks * (tb::kBK / p.a_box_ch);
    s.num_stages = (s.num_pieces + pps - 1) / pps;
  }
  if (t >= (1ll << 31)) return set_err(TIR_B200_ERR_UNSUPPORTED, "too many tiles");
  if (pieces > tb::kMaxPieces)
    return set_err(TIR_B200_ERR_UNSUPPORTED, "reduction too deep: %lld TMA pieces (max %d)",
                   static_cast<long long>(pieces), tb::kMaxPieces);
  p.total_pieces = static_cast<int32_t>(pieces);
  p.total_tiles = static_cast<int32_t>(t);
  return TIR_B200_OK;
}

// ------------------------------------------------------------------ split-K

// Split the reduction when the output tiles cannot fill half the machine: the
// ksplit CTAs of one output tile form a thread-block cluster and combine their
// fp32 partials through distributed shared memory in a fixed order
// (igemm.cuh cluster_reduce), then apply the whole epilogue — deterministic,
// no workspace, no memset, no atomics. <= 8 splits (portable cluster size).
int choose_ksplit(const tb::IgemmParams& p, int64_t out_tiles, int out_f16, int sms) {
  int nst_min = 1 << 30;
  for (int i = 0; i < p.num_sub; ++i) nst_min = std::min(nst_min, p.sub[i].num_stages);
  // every split needs >= 1 stage (an empty split would publish an unwritten accumulator)
  if (const int e = tb::options().ksplit) return std::max(1, std::min({8, e, nst_min}));
  // Fused-epilogue launches (the network graphs) are never split automatically:
  // one reduction order per output element whatever the batch, so a batch shard
  // is bit-identical to the same rows of the full-batch forward.
  if (out_f16 || p.bias || p.relu || p.residual) return 1;
  // At most half the SMs: the next launch's CTAs then enter on the other half while
  // this one runs, and their prologue is off the critical path (T2D: 64 CTAs 9.9 us,
  // 128 CTAs 10.6 us; tools/cta_timeline.py).
  if (out_tiles * 2 > sms / 2) return 1;
  int ks = static_cast<int>(std::min<int64_t>(sms / 2 / out_tiles, 8));
  ks = std::min(ks, nst_min / 2);  // at least two stages per split
  return std::max(ks, 1);
}


// ------------------------------------------------------------------ GMM

int gmm_impl(const uint16_t* A, const uint16_t* B, const float* Cin, void* C, int64_t M,
             int64_t N, int64_t K, int accumulate, int out_f16, const Epi& epi, cudaStream_t stream) {
  if (M < 0 || N < 0 || K < 0) return set_err(TIR_B200_ERR_VALUE, "gmm: negative extent");
  if (M == 0 || N == 0) return TIR_B200_OK;
  if (K == 0) {  // C = Cin (or 0): nothing to contract
    return set_err(TIR_B200_ERR_UNSUPPORTED, "gmm: K == 0");
  }
  if (!A || !B || !C || (accumulate && !Cin)) return set_err(TIR_B200_ERR_VALUE, "gmm: null operand");
  if (K % 8 || N % 8)
    return set_err(TIR_B200_ERR_UNSUPPORTED,
                   "gmm: K and N must be multiples of 8 (16-byte TMA row pitch); got K=%lld N=%lld",
                   static_cast<long long>(K), static_cast<long long>(N));
  if (M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 31))
    return set_err(TIR_B200_ERR_UNSUPPORTED, "gmm: extent too large");
  const DeviceInfo di = device_info();
  tb::IgemmParams p;
  std::memset(&p, 0, sizeof p);
  const int bn = choose_bn(N, (M + tb::kBM - 1) / tb::kBM, 1, (K + 15) / 16, di.sms, !out_f16 && !epi.on());
  const int ks = choose_ks(static_cast<int>((K + 63) / 64), 64, bn);
  const int ks_eff = bn >= 128 ? std::min(ks, 2) : ks;
  int rc = encode_2d(&p.tmA[0], A, M, K, 64, tb::kBM);
  if (rc) return rc;
  rc = encode_2d(&p.tmB, B, K, N, std::min(bn, 64), tb::kBK * ks_eff);
  if (rc) return rc;
  p.num_sub = 1;
  tb::SubProb& s = p.sub[0];
  set_sub_identity(s);
  s.m_count = static_cast<int32_t>(M);
  s.gx = static_cast<int32_t>(M);
  s.gy = s.gz = 1;
  s.num_pieces = static_cast<int32_t>((K + 63) / 64);
  p.groups = 1;
  p.a_mode = tb::A_TILED;
  p.a_box_ch = 64;
  p.cig = static_cast<int32_t>(K);
  p.cb_per_tap = s.num_pieces;
  p.b_mode = tb::B_STREAM;
  p.k_rows = static_cast<int32_t>(K);
  p.w_kx = p.w_ky = 1;
  p.cog = static_cast<int32_t>(N);
  p.ldy = static_cast<int32_t>(N);
  p.out_dims[0] = static_cast<int32_t>(M);
  p.out_dims[1] = p.out_dims[2] = 1;
  p.accumulate = accumulate;
  p.out_f16 = out_f16;
  p.Y = C;
  p.Yin = Cin;
  epi.apply(p);
  p.ksplit = 1;
  rc = finalize_tiles(p, bn, ks_eff);
  if (rc) return rc;
  p.ksplit = choose_ksplit(p, p.total_tiles, out_f16, di.sms);
  if (p.ksplit > 1) {
    rc = finalize_tiles(p, bn, ks_eff);
    if (rc) return rc;
  }
  if (p.ksplit == 1) {
    rc = pick_store_mode(p, bn, C, Cin, M, accumulate, out_f16);
    if (rc) return rc;
  }
  return launch_igemm(p, bn, ks_eff, stream);
}

// ------------------------------------------------------------------ batched GMM

int gmm_batched_impl(const uint16_t* A, int64_t a_rows, int64_t lda, const uint16_t* B, int64_t b_rows,
                     int64_t ldb, void* C, int64_t c_rows, int64_t ldc, int64_t M, int64_t N, int64_t K,
                     const tir_b200_batch_desc* bt, int out_f16, const Epi& epi, cudaStream_t stream) {
  if (!A || !B || !C || !bt) return set_err(TIR_B200_ERR_VALUE, "gmm_batched: null operand");
  if (M <= 0 || N <= 0 || K <= 0 || bt->z1n <= 0 || bt->z2n <= 0)
    return set_err(TIR_B200_ERR_VALUE, "gmm_batched: empty problem");
  if (M % tb::kBM || K % tb::kBK || N % 32)
    return set_err(TIR_B200_ERR_UNSUPPORTED, "gmm_batched: needs M %% 128 == 0, K %% 64 == 0, N %% 32 == 0");
  if (lda % 8 || ldb % 8 || ldc % 8)
    return set_err(TIR_B200_ERR_UNSUPPORTED, "gmm_batched: leading dims must be multiples of 8");
  if (epi.residual && !out_f16) return set_err(TIR_B200_ERR_UNSUPPORTED, "gmm_batched: residual needs fp16 C");
  // every problem's windows inside their tensors (checked at the z corners; coordinates are affine in z)
  const bool bkm = bt->b_kmajor != 0;
  const int64_t lim[3][2] = {{a_rows - M, lda - K}, {b_rows - (bkm ? N : K), ldb - (bkm ? K : N)},
                             {c_rows - M, ldc - N}};
  const int64_t* ax[3][2] = {{bt->a_row, bt->a_col}, {bt->b_row, bt->b_col}, {bt->c_row, bt->c_col}};
  for (int t = 0; t < 3; ++t)
    for (int d = 0; d < 2; ++d)
      for (int64_t z1 : {int64_t(0), bt->z1n - 1})
        for (int64_t z2 : {int64_t(0), bt->z2n - 1}) {
          const int64_t v = ax[t][d][0] + z1 * ax[t][d][1] + z2 * ax[t][d][2];
          if (v < 0 || v > lim[t][d] || v >= (1ll << 31))
            return set_err(TIR_B200_ERR_VALUE, "gmm_batched: operand %d window out of bounds", t);
        }
  const DeviceInfo di = device_info();
  tb::IgemmParams p;
  std::memset(&p, 0, sizeof p);
  int bn = 256;
  while (bn > 32 && N % bn) bn /= 2;
  const int64_t tiles_m = M / tb::kBM;
  const int64_t probs = bt->z1n * bt->z2n;
  while (bn > 32 && probs * tiles_m * (N / bn) < di.sms) bn /= 2;  // fill the machine
  const int ks = choose_ks(static_cast<int>(K / 64), 64, bn);
  const int ks_eff = bn >= 128 ? std::min(ks, 2) : ks;
  int rc = encode_2d(&p.tmA[0], A, a_rows, lda, 64, tb::kBM);
  if (rc) return rc;
  // MN-major B: boxes {min(BN, 64) cols, KS*64 rows}; K-major: {64 K, BN rows}
  rc = bkm ? encode_2d(&p.tmB, B, b_rows, ldb, 64, bn) : encode_2d(&p.tmB, B, b_rows, ldb, std::min(bn, 64), tb::kBK * ks_eff);
  if (rc) return rc;
  p.b_kmajor = bkm ? 1 : 0;
  p.num_sub = 1;
  tb::SubProb& s = p.sub[0];
  set_sub_identity(s);
  s.m_count = static_cast<int32_t>(M);
  s.gx = static_cast<int32_t>(M);
  s.gy = s.gz = 1;
  s.num_pieces = static_cast<int32_t>(K / 64);
  p.groups = 1;
  p.a_mode = tb::A_TILED;
  p.a_box_ch = 64;
  p.cig = static_cast<int32_t>(K);
  p.cb_per_tap = s.num_pieces;
  p.b_mode = tb::B_STREAM;
  p.k_rows = static_cast<int32_t>(b_rows);
  p.w_kx = p.w_ky = 1;
  p.cog = static_cast<int32_t>(N);
  p.ldy = static_cast<int32_t>(ldc);
  p.out_dims[0] = static_cast<int32_t>(M);
  p.out_dims[1] = p.out_dims[2] = 1;
  p.out_f16 = out_f16;
  p.Y = C;
  epi.apply(p);
  p.ksplit = 1;
  rc = finalize_tiles(p, bn, ks_eff);
  if (rc) return rc;
  p.batch_tiles = p.total_tiles;
  p.batch_z2 = static_cast<int32_t>(bt->z2n);
  if (static_cast<int64_t>(p.total_tiles) * probs >= (1ll << 31))
    return set_err(TIR_B200_ERR_UNSUPPORTED, "gmm_batched: too many tiles");
  p.total_tiles = static_cast<int32_t>(p.total_tiles * probs);
  auto axis = [](tb::BatchAxis& a, const int64_t* r, const int64_t* c) {
    for (int i = 0; i < 3; ++i) {
      a.row[i] = static_cast<int32_t>(r[i]);
      a.col[i] = static_cast<int32_t>(c[i]);
    }
  };
  axis(p.ba, bt->a_row, bt->a_col);
  axis(p.bb, bt->b_row, bt->b_col);
  axis(p.bc, bt->c_row, bt->c_col);
  // TMA-store epilogue over the whole C tensor (per-problem coordinates)
  rc = pick_store_mode(p, bn, C, nullptr, c_rows, 0, out_f16);
  if (rc) return rc;
  if (p.store_mode != 1) return set_err(TIR_B200_ERR_UNSUPPORTED, "gmm_batched: C must be 16-byte aligned");
  return launch_igemm(p, bn, ks_eff, stream);
}

// ------------------------------------------------------------------ conv (tensor cores)

int corner_limit(int rank) { return rank == 3 ? 32768 : rank == 4 ? 128 : 16; }
int offset_limit(int rank) { return rank == 3 ? 65536 : rank == 4 ? 256 : 32; }

// Im2col tensor map over X[N, (D,) (H,) W, C] (C contiguous).
int encode_im2col(CUtensorMap* m, const void* X, const Geo& g, int64_t c_total, int rank,
                  const int lower[3], const int upper[3], const int estride[3], int box_ch) {
  const Driver* d = driver();
  if (!d->im2col) return set_err(TIR_B200_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  // dims in TMA order: C, W, H, D, N (truncated to rank)
  cuuint64_t dims[5], strides[4];
  cuuint32_t estr[5];
  int lo[3], up[3];
  const int nsp = rank - 2;  // spatial dims used: W (, H (, D))
  dims[0] = static_cast<cuuint64_t>(c_total);
  estr[0] = 1;
  int64_t pitch = c_total * 2;
  for (int i = 0; i < nsp; ++i) {  // i=0:W, 1:H, 2:D  -> Geo index 2-i
    dims[1 + i] = static_cast<cuuint64_t>(g.in[2 - i]);
    strides[i] = static_cast<cuuint64_t>(pitch);
    pitch *= g.in[2 - i];
    estr[1 + i] = static_cast<cuuint32_t>(estride[2 - i]);
    lo[i] = lower[2 - i];
    up[i] = upper[2 - i];
  }
  // dims of unused spatial extents (must be 1) fold into the batch pitch
  for (int i = nsp; i < 3; ++i) pitch *= g.in[2 - i];
  dims[rank - 1] = static_cast<cuuint64_t>(g.n);
  strides[rank - 2] = static_cast<cuuint64_t>(pitch);
  estr[rank - 1] = 1;
  const int lim = corner_limit(rank);
  for (int i = 0; i < nsp; ++i)
    if (lo[i] < -lim || lo[i] >= lim || up[i] < -lim || up[i] >= lim)
      return set_err(TIR_B200_ERR_UNSUPPORTED, "conv: im2col corner out of range (%d, %d)", lo[i],
                     up[i]);
  CUresult r = d->im2col(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, static_cast<cuuint32_t>(rank),
                         const_cast<void*>(X), dims, strides, lo, up,
                         static_cast<cuuint32_t>(box_ch), static_cast<cuuint32_t>(tb::kBM), estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(box_ch * 2),
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(TIR_B200_ERR_CUDA, "cuTensorMapEncodeIm2col failed (%d)", static_cast<int>(r));
  // Same driver workaround CUTLASS applies to small im2col tensors (<= r580 drivers).
  const int64_t bytes = g.n * g.in[0] * g.in[1] * g.in[2] * c_total * 2;
  if (d->version <= 13010 && bytes < 131072) reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
  return TIR_B200_OK;
}

int pick_box(int64_t cig) {
  for (int b : {64, 32, 16, 8})
    if (cig % b == 0) return b;
  return 0;
}

// ------------------------------------------------------------------ conv (halo, stride 1)


template <int BN, int KH, int KW>
int launch_halo_bn(tb::HaloParams& p, cudaStream_t stream) {
  using Cfg = tb::HaloCfg<BN>;
  const DeviceInfo di = device_info();
  const int keys = p.groups * p.tiles_n;
  if (keys > di.sms) return kNotEligible;
  if (BN > 64 && p.b_rows * Cfg::kBRowBytes >= (1 << 18)) return kNotEligible;
  const int fixed = 1024 + 256 + p.b_rows * BN * 2 + 2 * p.stage_bytes;
  const int slab = p.slab_rows * 128;
  const int stages = std::min(4, (di.smem_optin - fixed) / slab);
  if (stages < 2) return kNotEligible;
  p.stages = stages;
  const size_t smem = Cfg::smem_bytes(p.stages, p.slab_rows, p.b_rows, p.stage_bytes);
  CUDA_TRY(ensure_smem(tb::conv_halo_kernel<BN, KH, KW>, smem));
  int grid = std::min(p.total_tiles, di.sms / keys * keys);
  if (const int e = tb::options().max_ctas) grid = std::max(1, std::min(grid, e));
  p.trace = g_trace;
  p.l2_prefetch = tb::options().l2_prefetch;
  CUDA_TRY(launch_pdl(tb::conv_halo_kernel<BN, KH, KW>, grid, tb::kHaloThreads, smem, stream, p));
  ++g_launches;
  return TIR_B200_OK;
}

// Stride-1 2-D convolution as halo tiles (see halo.cuh). Returns kNotEligible
// for shapes outside its envelope.
int conv_halo_impl(const Geo& g, const uint16_t* X, const uint16_t* W, const float* Yin, void* Y,
                   int accumulate, int out_f16, const Epi& epi, cudaStream_t stream) {
  if (tb::options().no_halo) return kNotEligible;
  if (g.transposed || g.in[0] != 1 || g.k[0] != 1 || g.p[0] != 0) return kNotEligible;
  if (g.s[1] != 1 || g.s[2] != 1 || g.d[1] != g.d[2]) return kNotEligible;
  const int64_t cig = g.ci / g.g, cog = g.co / g.g;
  if (cig % 64 || g.co % 8) return kNotEligible;
  if (accumulate && !Yin) return kNotEligible;
  const int64_t d = g.d[1], KH = g.k[1], KW = g.k[2];
  const int64_t OH = g.out[1], OW = g.out[2];
  int64_t Wt, R;
  if (OW + (KW - 1) * d <= 128) {
    Wt = OW;
    R = 128 / (OW + (KW - 1) * d);
  } else {
    Wt = 128 - (KW - 1) * d;
    R = 1;
    if (Wt < 16) return kNotEligible;
  }
  const int64_t Wv = Wt + (KW - 1) * d;
  int64_t HR = R + (KH - 1) * d;
  const int64_t max_off = (KH - 1) * d * Wv + (KW - 1) * d;
  if (Wv > 256 || HR > 256) return kNotEligible;
  int64_t slab_rows = std::max(HR * Wv, max_off + 128);
  slab_rows = (slab_rows + 7) / 8 * 8;
  if (slab_rows > tb::kHaloMaxRows) return kNotEligible;
  const int64_t taps = KH * KW;
  const DeviceInfo di = device_info();

  tb::HaloParams p;
  std::memset(&p, 0, sizeof p);
  p.n = static_cast<int32_t>(g.n);
  p.oh = static_cast<int32_t>(OH);
  p.ow = static_cast<int32_t>(OW);
  p.co = static_cast<int32_t>(g.co);
  p.cig = static_cast<int32_t>(cig);
  p.cog = static_cast<int32_t>(cog);
  p.groups = static_cast<int32_t>(g.g);
  p.kh = static_cast<int32_t>(KH);
  p.kw = static_cast<int32_t>(KW);
  p.dil = static_cast<int32_t>(d);
  p.pad_h = static_cast<int32_t>(g.p[1]);
  p.pad_w = static_cast<int32_t>(g.p[2]);
  p.R = static_cast<int32_t>(R);
  p.Wt = static_cast<int32_t>(Wt);
  p.Wv = static_cast<int32_t>(Wv);
  p.HR = static_cast<int32_t>(HR);
  p.tiles_w = static_cast<int32_t>((OW + Wt - 1) / Wt);
  p.tiles_h = static_cast<int32_t>((OH + R - 1) / R);
  p.cblocks = static_cast<int32_t>(cig / 64);
  p.b_rows = static_cast<int32_t>(taps * cig);
  p.slab_rows = static_cast<int32_t>(slab_rows);
  p.accumulate = accumulate;
  p.out_f16 = out_f16;
  p.Y = Y;
  p.Yin = Yin;
  p.bias = epi.bias;
  p.relu = epi.relu;
  p.residual = epi.residual;
  // N tile: whole group width up to 256 when that still fills the machine.
  const int64_t spatial_tiles = g.n * p.tiles_h * p.tiles_w;
  const int bn = choose_bn(cog, spatial_tiles, g.g, taps * (cig / 16), di.sms, !out_f16 && !epi.on());
  p.tiles_n = static_cast<int32_t>((cog + bn - 1) / bn);
  const int64_t total = spatial_tiles * g.g * p.tiles_n;
  if (total >= (1ll << 31)) return kNotEligible;
  p.total_tiles = static_cast<int32_t>(total);
  // X as 4-D [N, H, W, C] (C fastest), box {64, Wv, HR, 1}; OOB -> zero padding
  {
    const Driver* drv = driver();
    if (!drv->tiled) return set_err(TIR_B200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.ci), static_cast<cuuint64_t>(g.in[2]),
                          static_cast<cuuint64_t>(g.in[1]), static_cast<cuuint64_t>(g.n)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.ci * 2),
                             static_cast<cuuint64_t>(g.ci * 2 * g.in[2]),
                             static_cast<cuuint64_t>(g.ci * 2 * g.in[2] * g.in[1])};
    cuuint32_t box[4] = {64, static_cast<cuuint32_t>(Wv), static_cast<cuuint32_t>(HR), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = drv->tiled(&p.tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<uint16_t*>(X), dims,
                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(TIR_B200_ERR_CUDA, "halo X tensor map failed (%d)", (int)r);
  }
  p.b_box_rows = 64;
  for (int rows : {256, 192, 128}) {
    if (p.b_rows % rows == 0) {
      p.b_box_rows = rows;
      break;
    }
  }
  int rc = encode_2d(&p.tmW, W, taps * cig, g.co, std::min(bn, 64), p.b_box_rows);
  if (rc) return rc;
  // Epilogue: TMA bulk stores of [R][Wt][32] boxes when a 32-column chunk never
  // crosses a group (cog % 32 == 0 or a single group) and, for accumulate, Y is
  // updated in place (reduce-add). Otherwise direct register stores.
  p.store_mode = 0;
  p.stage_bytes = 0;
  if (bn >= 32 && (g.g == 1 || cog % 32 == 0) && (!accumulate || (Yin == Y && !epi.on())) &&
      !tb::options().no_tma_store) {
    const Driver* drv = driver();
    const int esz = out_f16 ? 2 : 4;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.co), static_cast<cuuint64_t>(OW),
                          static_cast<cuuint64_t>(OH), static_cast<cuuint64_t>(g.n)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.co * esz),
                             static_cast<cuuint64_t>(g.co * esz * OW),
                             static_cast<cuuint64_t>(g.co * esz * OW * OH)};
    cuuint32_t box[4] = {32, static_cast<cuuint32_t>(Wt), static_cast<cuuint32_t>(R), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = drv->tiled(&p.tmY, out_f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                            4, Y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            out_f16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) {
      p.store_mode = accumulate ? 2 : 1;
      p.stage_bytes = static_cast<int32_t>((R * Wt * 32 * esz + 1023) / 1024 * 1024);
    }
  }
  const bool k3 = KH == 3 && KW == 3;
  switch (bn) {
    case 16: return k3 ? launch_halo_bn<16, 3, 3>(p, stream) : launch_halo_bn<16, 0, 0>(p, stream);
    case 32: return k3 ? launch_halo_bn<32, 3, 3>(p, stream) : launch_halo_bn<32, 0, 0>(p, stream);
    case 64: return k3 ? launch_halo_bn<64, 3, 3>(p, stream) : launch_halo_bn<64, 0, 0>(p, stream);
    case 128: return k3 ? launch_halo_bn<128, 3, 3>(p, stream) : launch_halo_bn<128, 0, 0>(p, stream);
    case 256: return k3 ? launch_halo_bn<256, 3, 3>(p, stream) : launch_halo_bn<256, 0, 0>(p, stream);
  }
  return kNotEligible;
}

// ------------------------------------------------------------------ conv (rowpack, CI = 3 stems)

template <int BN, int KH, int KW, int CI, int DW, bool D3>
int launch_rowpack_k(tb::RowpackParams& p, size_t smem, cudaStream_t stream) {
  CUDA_TRY(ensure_smem(tb::conv_rowpack_kernel<BN, KH, KW, CI, DW, D3>, smem));
  const DeviceInfo di = device_info();
  const int grid = std::min(p.total_units, di.sms);
  p.trace = g_trace;
  CUDA_TRY(launch_pdl(tb::conv_rowpack_kernel<BN, KH, KW, CI, DW, D3>, grid, tb::kRpThreads, smem, stream, p));
  ++g_launches;
  return TIR_B200_OK;
}

template <int BN, int KH, int KW, int CI, int DW>
int launch_rowpack(tb::RowpackParams& p, size_t smem, cudaStream_t stream, bool d3) {
  return d3 ? launch_rowpack_k<BN, KH, KW, CI, DW, true>(p, smem, stream)
            : launch_rowpack_k<BN, KH, KW, CI, DW, false>(p, smem, stream);
}

// Small-channel convolutions whose (kh, kw, c) window fits one TMEM K vector
// (rowpack.cuh): the C3D paper shape and the CI = 3 network stems. Returns
// kNotEligible outside its envelope (the im2col path takes those).
int conv_rowpack_impl(const Geo& g, const uint16_t* X, const uint16_t* W, const float* Yin, void* Y,
                      int accumulate, int out_f16, const Epi& epi, cudaStream_t stream) {
  if (tb::options().no_rowpack) return kNotEligible;
  if (g.transposed || g.g != 1 || epi.residual) return kNotEligible;
  if (g.co != 64 && g.co != 32) return kNotEligible;
  if ((g.s[2] * g.ci) % 2) return kNotEligible;  // every lane's window starts at the same element parity
  if (accumulate && epi.on()) return kNotEligible;  // the C-ABI order is (Yin + acc) + bias: not a reduce-add
  if (accumulate && Yin != Y) return kNotEligible;  // in-place accumulate = TMA reduce-add
  const int64_t kwc = g.k[2] * g.ci;
  const int64_t wpk = (kwc + 1) / 2;
  const int64_t KH = g.k[1];
  const int64_t span = (g.k[2] - 1) * g.d[2] * g.ci + g.ci;  // window elements first to last
  // instantiated windows (KH x KW x CI, w-dilation): 7x7x3 (C3D, ResNet stem), 7x7x3 d2 (DIL), 3x3x3 (MobileNet stem)
  const int shape = (g.ci == 3 && KH == 7 && g.k[2] == 7 && g.d[2] == 1) ? 0
                    : (g.ci == 3 && KH == 7 && g.k[2] == 7 && g.d[2] == 2) ? 1
                    : (g.ci == 3 && KH == 3 && g.k[2] == 3 && g.d[2] == 1) ? 2 : -1;
  if (shape < 0) return kNotEligible;
  const int64_t kwords = (KH * wpk + 7) / 8 * 8;
  const int64_t kp = 2 * kwords;
  const int64_t OD = g.out[0], OH = g.out[1], OW = g.out[2];
  const int64_t Wt = std::min<int64_t>(16, OW);
  const int64_t R = 128 / Wt;
  // TMA box starts are 16-byte aligned in the innermost dim: the box begins `shift`
  // elements before the tile's first input element (the same shift for every tile
  // column when Wt*sw*CI % 8 == 0); runs starting at odd elements are funnel-shifted
  const int64_t tiles_w0 = (OW + Wt - 1) / Wt;
  if (tiles_w0 > 1 && (Wt * g.s[2] * g.ci) % 8) return kNotEligible;
  const int64_t shift = (8 - (g.p[2] * g.ci) % 8) % 8;
  int64_t box_w = (shift + (Wt - 1) * g.s[2] * g.ci + span + 2 + 7) / 8 * 8;
  // A warp's lanes cover two tile rows (Wt = 16): a row step of 16 (mod 32) words
  // keeps the builders' 32-bit shared loads conflict-free (lane c reads word 3c + ...)
  for (int64_t b = box_w; b <= box_w + 56 && b <= 256; b += 8) {
    if (Wt == 16 && (g.s[1] * b / 2) % 32 == 16) {
      box_w = b;
      break;
    }
  }
  const int64_t box_h = (R - 1) * g.s[1] + (KH - 1) * g.d[1] + 1;
  if (box_w > 256 || box_h > 256) return kNotEligible;
  const int64_t wci = g.in[2] * g.ci;
  if ((wci * 2) % 16) return kNotEligible;  // TMA row pitch
  // TMEM rings: ceil(KD/sd) depths in flight + one draining (>= 2: the epilogue of a
  // tile overlaps the next tile's MMAs), then as many A buffers as fit (the builders
  // run ahead of the MMAs by nabuf - 1 planes)
  if (g.d[0] != 1) return kNotEligible;
  const bool d3 = g.k[0] > 1;  // 3-D: a ring of kRpMaxSlots depth accumulators (rowpack.cuh)
  if (d3 && (g.k[0] + g.s[0] - 1) / g.s[0] + 1 > tb::kRpMaxSlots) return kNotEligible;
  const DeviceInfo di = device_info();
  const int bn = static_cast<int>(g.co);
  const int64_t b_bytes = g.k[0] * kp * bn * 2;
  const int stage_bytes = static_cast<int>((R * Wt * 32 * (out_f16 ? 2 : 4) + 1023) / 1024 * 1024);
  const int slot_bytes = static_cast<int>((box_w * box_h * 2 + 1023) / 1024 * 1024);
  const int64_t fixed = 1024 + b_bytes + 2 * stage_bytes + 256 + 16 * 3 * 16 + 16;  // + plane-descriptor ring
  // deep raw ring: each plane's box is a latency-bound handful of short DRAM rows
  const int stages = static_cast<int>(std::min<int64_t>(8, (di.smem_optin - fixed) / slot_bytes));
  if (stages < 2) return kNotEligible;
  const size_t smem = static_cast<size_t>(fixed + static_cast<int64_t>(stages) * slot_bytes);
  const int64_t tiles_h = (OH + R - 1) / R, tiles_w = (OW + Wt - 1) / Wt;
  const int64_t units = g.n * tiles_h * tiles_w;  // a unit: one spatial tile through the whole depth
  if (units >= (1ll << 31) || g.n * g.in[0] >= (1ll << 31)) return kNotEligible;

  // packed weight panel [KD * Kp, CO] in the per-stream workspace
  void* ws = nullptr;
  int rc = workspace(static_cast<size_t>(b_bytes) + 256, stream, &ws);
  if (rc) return rc;
  uint16_t* Bp = static_cast<uint16_t*>(ws);
  tb::pack_rowpack_weights_kernel<<<tb::grid_for(g.k[0] * kp * bn), 256, 0, stream>>>(
      W, Bp, static_cast<int32_t>(g.k[0]), static_cast<int32_t>(KH), static_cast<int32_t>(g.k[2]),
      static_cast<int32_t>(g.ci), bn, static_cast<int32_t>(wpk), static_cast<int32_t>(kp));
  CUDA_TRY(cudaGetLastError());
  ++g_launches;

  tb::RowpackParams p;
  std::memset(&p, 0, sizeof p);
  const Driver* drv = driver();
  if (!drv->tiled) return set_err(TIR_B200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  {  // X as 3-D [N*D, H, W*CI]: box {box_w, box_h, 1}; OOB -> zero padding
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(wci), static_cast<cuuint64_t>(g.in[1]),
                          static_cast<cuuint64_t>(g.n * g.in[0])};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(wci * 2), static_cast<cuuint64_t>(wci * 2 * g.in[1])};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = drv->tiled(&p.tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<uint16_t*>(X), dims, strides,
                            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(TIR_B200_ERR_CUDA, "rowpack X tensor map failed (%d)", (int)r);
  }
  {  // packed weights [KD*Kp, CO]: one box of Kp rows per kd
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(bn), static_cast<cuuint64_t>(g.k[0] * kp)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(bn * 2)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(bn), static_cast<cuuint32_t>(kp)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = drv->tiled(&p.tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, Bp, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            bn == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(TIR_B200_ERR_CUDA, "rowpack W tensor map failed (%d)", (int)r);
  }
  {  // Y as 4-D [N*OD, OH, OW, CO]: box {32, Wt, R, 1}
    const int esz = out_f16 ? 2 : 4;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.co), static_cast<cuuint64_t>(OW), static_cast<cuuint64_t>(OH),
                          static_cast<cuuint64_t>(g.n * OD)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.co * esz), static_cast<cuuint64_t>(g.co * esz * OW),
                             static_cast<cuuint64_t>(g.co * esz * OW * OH)};
    cuuint32_t box[4] = {32, static_cast<cuuint32_t>(Wt), static_cast<cuuint32_t>(R), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = drv->tiled(&p.tmY, out_f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                            Y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            out_f16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(TIR_B200_ERR_CUDA, "rowpack Y tensor map failed (%d)", (int)r);
  }
  p.n = static_cast<int32_t>(g.n);
  p.d = static_cast<int32_t>(g.in[0]);
  p.ci = static_cast<int32_t>(g.ci);
  p.od = static_cast<int32_t>(OD);
  p.oh = static_cast<int32_t>(OH);
  p.ow = static_cast<int32_t>(OW);
  p.kd = static_cast<int32_t>(g.k[0]);
  p.sd = static_cast<int32_t>(g.s[0]);
  p.sh = static_cast<int32_t>(g.s[1]);
  p.sw = static_cast<int32_t>(g.s[2]);
  p.pd = static_cast<int32_t>(g.p[0]);
  p.ph = static_cast<int32_t>(g.p[1]);
  p.pw = static_cast<int32_t>(g.p[2]);
  p.dd = static_cast<int32_t>(g.d[0]);
  p.dh = static_cast<int32_t>(g.d[1]);
  p.R = static_cast<int32_t>(R);
  p.Wt = static_cast<int32_t>(Wt);
  p.tiles_h = static_cast<int32_t>(tiles_h);
  p.tiles_w = static_cast<int32_t>(tiles_w);
  p.total_units = static_cast<int32_t>(units);
  p.kp = static_cast<int32_t>(kp);
  p.box_w = static_cast<int32_t>(box_w);
  p.box_h = static_cast<int32_t>(box_h);
  p.shift = static_cast<int32_t>(shift);
  p.stages = stages;
  p.slot_bytes = slot_bytes;
  p.out_f16 = out_f16;
  p.store_mode = accumulate ? 2 : 1;
  p.stage_bytes = stage_bytes;
  p.debug = tb::options().rowpack_debug;
  p.backoff_ns = tb::options().rp_backoff;
  p.backoff_ns2 = tb::options().rp_backoff2;
  p.bias = epi.bias;
  p.act = epi.relu;
  if (bn == 64) {
    if (shape == 0) return launch_rowpack<64, 7, 7, 3, 1>(p, smem, stream, d3);
    if (shape == 1) return launch_rowpack<64, 7, 7, 3, 2>(p, smem, stream, d3);
    return launch_rowpack<64, 3, 3, 3, 1>(p, smem, stream, d3);
  }
  if (shape == 0) return launch_rowpack<32, 7, 7, 3, 1>(p, smem, stream, d3);
  if (shape == 1) return launch_rowpack<32, 7, 7, 3, 2>(p, smem, stream, d3);
  return launch_rowpack<32, 3, 3, 3, 1>(p, smem, stream, d3);
}

int conv_tc_impl(const Geo& g0, const uint16_t* X0, const uint16_t* W0, const float* Yin, void* Y,
                 int accumulate, int out_f16, const Epi& epi, cudaStream_t stream) {
  Geo g = g0;
  const uint16_t* X = X0;
  const uint16_t* W = W0;
  int64_t cig = g.ci / g.g;
  const int64_t cog = g.co / g.g;
  int64_t taps = g.k[0] * g.k[1] * g.k[2];
  // Small-channel layers whose KH x KW window is large (C3D / DIL 7x7 x CI=3 =
  // 147 values): pack (kh, kw, c) into 64-aligned channels (pack_hw, prep.cuh);
  // what remains is a depth-only (C3D) or 1x1 (DIL) conv streaming 64-channel
  // im2col pieces. Bit-exact relayout. Opt-in (TIR_B200_PACK_HW=1): measured on
  // B200 the 6.4x larger relayout (1.23 GB for the C3D paper shape, written and
  // read back through HBM) costs more than the request-bound 32-channel pieces
  // it removes (C3D 1260 vs 724 us).
  // Default when the (kh, kw, c) relayout is no bigger than 1.5x the (kw, c) one
  // (e.g. MobileNet-V2's 3x3 stem: 27 -> 32 channels, the same bytes as the
  // (kw, c) form, and the conv becomes a 1x1 GEMM instead of 16-channel pieces).
  const int64_t hw_cp = (g.k[1] * g.k[2] * cig + 63) / 64 * 64 <= 32 ? 32 : (g.k[1] * g.k[2] * cig + 63) / 64 * 64;
  const int64_t kw_cp = g.k[2] * cig <= 8 ? 8 : g.k[2] * cig <= 16 ? 16 : g.k[2] * cig <= 32 ? 32 : 64;
  const bool hw_small = g.out[1] * hw_cp * 2 <= 3 * g.in[1] * kw_cp;  // per output column, per image row block
  if (cig % 8 && g.g == 1 && !g.transposed && g.k[1] > 1 && g.k[1] * g.k[2] * cig <= 256 &&
      (tb::options().pack_hw == 1 || (hw_small && tb::options().pack_hw != 0))) {
    const int64_t cp = hw_cp;
    const int64_t rows = g.n * g.in[0] * g.out[1];
    const size_t xbytes = static_cast<size_t>(rows * g.out[2] * cp * 2);
    const size_t wbytes = static_cast<size_t>(g.k[0] * cp * g.co * 2);
    void* ws = nullptr;
    int rc = workspace(xbytes + wbytes + 512, stream, &ws);
    if (rc) return rc;
    uint16_t* Xp = static_cast<uint16_t*>(ws);
    uint16_t* Wp = reinterpret_cast<uint16_t*>(static_cast<char*>(ws) + (xbytes + 255) / 256 * 256);
    const int prc = tb::launch_pack_hw(X, Xp, W, Wp, rows, g.in[1], g.in[2], cig, g.out[1], g.out[2], g.k[1], g.k[2],
                                       g.s[1], g.s[2], g.p[1], g.p[2], g.d[1], g.d[2], cp, g.k[0], g.co, stream);
    if (prc == 1) return set_err(TIR_B200_ERR_CUDA, "pack kernel launch failed");
    if (prc == 0) {
      ++g_launches;
      X = Xp;
      W = Wp;
      g.in[1] = g.out[1];
      g.in[2] = g.out[2];
      g.ci = cp;
      for (int i = 1; i < 3; ++i) {
        g.k[i] = 1;
        g.s[i] = 1;
        g.p[i] = 0;
        g.d[i] = 1;
      }
      cig = cp;
      taps = g.k[0];
    }
  }
  // Small-channel layers (CI = 3 in C3D / DIL): pack the KW taps into the
  // channel dim ((kw, c) packing, prep.cuh) so each im2col piece carries
  // KW*CI real channels instead of CI padded to 8. Bit-exact relayout.
  if (cig % 8 && g.g == 1 && !g.transposed && g.k[2] > 1 && g.k[2] * cig <= 64 &&
      tb::options().pack_kw) {
    const int64_t kwc = g.k[2] * cig;
    const int64_t cp = kwc <= 8 ? 8 : kwc <= 16 ? 16 : kwc <= 32 ? 32 : 64;
    const int64_t rows = g.n * g.in[0] * g.in[1];
    const int64_t khd = g.k[0] * g.k[1];
    const size_t xbytes = static_cast<size_t>(rows * g.out[2] * cp * 2);
    const size_t wbytes = static_cast<size_t>(khd * cp * g.co * 2);
    void* ws = nullptr;
    int rc = workspace(xbytes + wbytes + 512, stream, &ws);
    if (rc) return rc;
    uint16_t* Xp = static_cast<uint16_t*>(ws);
    uint16_t* Wp = reinterpret_cast<uint16_t*>(static_cast<char*>(ws) + (xbytes + 255) / 256 * 256);
    const int prc = tb::launch_pack_kw_fused(X, Xp, W, Wp, rows, g.in[2], cig, g.out[2], g.k[2], g.s[2], g.p[2],
                                             g.d[2], cp, khd, kwc, g.co, stream);
    if (prc == 1) return set_err(TIR_B200_ERR_CUDA, "pack kernel launch failed");
    if (prc == 0) {
      ++g_launches;
    } else {  // rows too long for the staged kernel: the two generic relayout kernels
      if (tb::launch_pack_kw(X, Xp, rows, g.in[2], cig, g.out[2], g.k[2], g.s[2], g.p[2], g.d[2], cp, stream))
        return set_err(TIR_B200_ERR_CUDA, "pack kernel launch failed");
      ++g_launches;
      if (tb::launch_pack_kw_weights(W, Wp, khd, kwc, cp, g.co, stream))
        return set_err(TIR_B200_ERR_CUDA, "pack kernel launch failed");
      ++g_launches;
    }
    X = Xp;
    W = Wp;
    g.in[2] = g.out[2];
    g.ci = cp;
    g.k[2] = 1;
    g.s[2] = 1;
    g.p[2] = 0;
    g.d[2] = 1;
    cig = cp;
    taps = g.k[0] * g.k[1];
  }
  // Channel padding (a bit-exact layout step): TMA needs a 16-byte pixel pitch.
  // Channels are group-major, so padding each group's CI/G block is the same
  // kernel over pixels x groups rows; weights pad their CI/G rows per tap.
  if (cig % 8) {
    const int64_t cip = (cig + 7) / 8 * 8;
    const int64_t pix = g.n * g.in[0] * g.in[1] * g.in[2] * g.g;
    const size_t xbytes = static_cast<size_t>(pix * cip * 2);
    const size_t wbytes = static_cast<size_t>(taps * cip * g.co * 2);
    void* ws = nullptr;
    int rc = workspace(xbytes + wbytes + 256, stream, &ws);
    if (rc) return rc;
    uint16_t* Xp = static_cast<uint16_t*>(ws);
    uint16_t* Wp = reinterpret_cast<uint16_t*>(static_cast<char*>(ws) + (xbytes + 255) / 256 * 256);
    rc = tb::launch_pad_channels(X, Xp, pix, cig, cip, stream);
    if (rc) return set_err(TIR_B200_ERR_CUDA, "pad kernel launch failed");
    ++g_launches;
    rc = tb::launch_pad_weight_rows(W, Wp, taps, cig, cip, g.co, stream);
    if (rc) return set_err(TIR_B200_ERR_CUDA, "pad kernel launch failed");
    ++g_launches;
    X = Xp;
    W = Wp;
    g.ci = cip * g.g;
    cig = cip;
  }
  const int box = pick_box(cig);
  if (!box) return set_err(TIR_B200_ERR_UNSUPPORTED, "conv: channels per group %lld", (long long)cig);
  if (g.co % 8) return set_err(TIR_B200_ERR_UNSUPPORTED, "conv: CO must be a multiple of 8");
  // Spatial rank of the TMA view.
  int rank = 5;
  if (g.in[0] == 1 && g.k[0] == 1 && g.p[0] == 0 && g.s[0] == 1) {
    rank = (g.in[1] == 1 && g.k[1] == 1 && g.p[1] == 0 && g.s[1] == 1) ? 3 : 4;
  }
  const int nsp = rank - 2;
  auto used = [&](int i) { return i >= 3 - nsp; };  // Geo index i (0=D,1=H,2=W)

  const DeviceInfo di = device_info();
  tb::IgemmParams p;
  std::memset(&p, 0, sizeof p);
  p.groups = static_cast<int32_t>(g.g);
  p.a_mode = rank;
  p.a_box_ch = box;
  p.cig = static_cast<int32_t>(cig);
  p.cb_per_tap = static_cast<int32_t>(cig / box);
  p.k_rows = static_cast<int32_t>(taps * cig);
  p.w_kx = static_cast<int32_t>(g.k[2]);
  p.w_ky = static_cast<int32_t>(g.k[1]);
  p.cog = static_cast<int32_t>(cog);
  p.ldy = static_cast<int32_t>(g.co);
  p.out_dims[0] = static_cast<int32_t>(g.out[2]);
  p.out_dims[1] = static_cast<int32_t>(g.out[1]);
  p.out_dims[2] = static_cast<int32_t>(g.out[0]);
  p.accumulate = accumulate;
  p.out_f16 = out_f16;
  p.Y = Y;
  p.Yin = Yin;
  // Group packing (igemm.cuh GP): 64 / cig groups of 16 or 32 input channels share
  // one 64-channel im2col piece per tap (one TMA request instead of 64 / cig narrow
  // ones), each group an N = 32 MMA into its own accumulator columns.
  int gp = 1;
  if (!g.transposed && g.g > 1 && (cig == 16 || cig == 32) && cog == 32 && g.g % (64 / cig) == 0 &&
      taps * cig <= 256 && !tb::options().no_gpack)
    gp = static_cast<int>(64 / cig);
  if (gp > 1) {
    p.groups = static_cast<int32_t>(g.g / gp);
    p.a_box_ch = 64;
    p.cig = 64;
    p.cb_per_tap = 1;
    p.k_rows = static_cast<int32_t>(taps * 64);
    p.cog = 32 * gp;
    p.gp_taps = static_cast<int32_t>(taps);
    p.gp_kpg = static_cast<int32_t>(cig / 16);
  }
  epi.apply(p);

  const int lim_off = offset_limit(rank);
  if (!g.transposed) {
    p.num_sub = 1;
    tb::SubProb& s = p.sub[0];
    set_sub_identity(s);
    int lower[3], upper[3], estr[3];
    for (int i = 0; i < 3; ++i) {
      lower[i] = used(i) ? static_cast<int>(-g.p[i]) : 0;
      upper[i] = used(i) ? static_cast<int>(g.p[i] - g.d[i] * (g.k[i] - 1)) : 0;
      estr[i] = used(i) ? static_cast<int>(g.s[i]) : 1;
      if (used(i) && (g.k[i] - 1) * g.d[i] >= lim_off)
        return set_err(TIR_B200_ERR_UNSUPPORTED, "conv: dilated kernel extent exceeds im2col offsets");
      if (used(i) && g.s[i] > 8)
        return set_err(TIR_B200_ERR_UNSUPPORTED, "conv: stride > 8");
    }
    const int64_t M = g.n * g.out[0] * g.out[1] * g.out[2];
    if (M >= (1ll << 31)) return set_err(TIR_B200_ERR_UNSUPPORTED, "conv: too many output pixels");
    s.m_count = static_cast<int32_t>(M);
    s.gx = static_cast<int32_t>(g.out[2]);
    s.gy = static_cast<int32_t>(g.out[1]);
    s.gz = static_cast<int32_t>(g.out[0]);
    for (int i = 0; i < 3; ++i) {  // SubProb index 0=x(W),1=y(H),2=z(D) <- Geo 2-i
      s.a_lo[i] = lower[2 - i];
      s.a_st[i] = static_cast<int32_t>(g.s[2 - i]);
      s.taps[i] = static_cast<int32_t>(g.k[2 - i]);
      s.a_dil[i] = static_cast<int32_t>(g.d[2 - i]);
    }
    s.num_pieces = static_cast<int32_t>(taps * p.cb_per_tap);
    p.b_mode = tb::B_STREAM;
    int rc = encode_im2col(&p.tmA[0], X, g, g.ci, rank, lower, upper, estr, p.a_box_ch);
    if (rc) return rc;
    const int bn = gp > 1 ? p.cog
                          : choose_bn(cog, (M + tb::kBM - 1) / tb::kBM, g.g, taps * ((cig + 15) / 16), di.sms,
                                      !out_f16 && !epi.on());
    int ks = choose_ks(s.num_pieces, p.a_box_ch, bn);
    if (bn >= 128) ks = std::min(ks, 2);
    // GP: B is read as each packed group's [taps*cig, 32] block, one box per group
    rc = gp > 1 ? encode_2d(&p.tmB, W, taps * cig, g.co, 32, static_cast<int>(taps * cig))
                : encode_2d(&p.tmB, W, taps * cig, g.co, std::min(bn, 64), tb::kBK * ks);
    if (rc) return rc;
    p.ksplit = 1;
    rc = finalize_tiles(p, bn, ks);
    if (rc) return rc;
    if (gp > 1) {
      rc = pick_store_mode(p, bn, Y, Yin, M, accumulate, out_f16);
      if (rc) return rc;
      rc = launch_igemm_gp(p, bn, ks, stream);
      if (rc != kNotEligible) return rc;
      return set_err(TIR_B200_ERR_UNSUPPORTED, "grouped conv: packed plan does not fit");
    }
    p.ksplit = choose_ksplit(p, p.total_tiles, out_f16, di.sms);
    if (p.ksplit > 1) {
      rc = finalize_tiles(p, bn, ks);
      if (rc) return rc;
    }
    if (p.ksplit == 1) {
      rc = pick_store_mode(p, bn, Y, Yin, M, accumulate, out_f16);
      if (rc) return rc;
    }
    return launch_igemm(p, bn, ks, stream);
  }

  // Transposed (T2D): sub-pixel decomposition into prod(s) stride-1 convs, one
  // per output parity class q: o = s*a + q, taps k = r0 + s*t (r0 = (q+p) mod s),
  // input i = a + c - t (c = (q+p) div s). Flipping t makes each class a forward
  // correlation with lower corner c - (T-1); the epilogue scatters rows to o.
  if (g.g != 1) return set_err(TIR_B200_ERR_UNSUPPORTED, "T2D: groups must be 1");
  for (int i = 0; i < 3; ++i)
    if (g.d[i] != 1) return set_err(TIR_B200_ERR_UNSUPPORTED, "T2D: dilation must be 1");
  const int nclass = static_cast<int>(g.s[0] * g.s[1] * g.s[2]);
  if (nclass > tb::kMaxSub)
    return set_err(TIR_B200_ERR_UNSUPPORTED, "T2D: %d sub-pixel classes (max %d)", nclass, tb::kMaxSub);
  p.b_mode = tb::B_PIECES;
  int64_t m_max = 0;
  int ns = 0;
  for (int qd = 0; qd < g.s[0]; ++qd)
    for (int qh = 0; qh < g.s[1]; ++qh)
      for (int qw = 0; qw < g.s[2]; ++qw) {
        const int q[3] = {qd, qh, qw};
        int lower[3], upper[3], estr[3] = {1, 1, 1};
        int T[3], A[3], base[3], step[3];
        bool empty = false;
        for (int i = 0; i < 3; ++i) {
          const int64_t s_ = g.s[i], p_ = g.p[i], k_ = g.k[i];
          const int64_t r0 = (q[i] + p_) % s_;
          const int64_t c = (q[i] + p_) / s_;
          T[i] = k_ > r0 ? static_cast<int>((k_ - r0 + s_ - 1) / s_) : 0;
          A[i] = g.out[i] > q[i] ? static_cast<int>((g.out[i] - q[i] + s_ - 1) / s_) : 0;
          if (T[i] == 0 || A[i] == 0) empty = true;
          lower[i] = static_cast<int>(c - (T[i] - 1));
          upper[i] = static_cast<int>(A[i] - g.in[i] + lower[i]);
          base[i] = static_cast<int>(r0 + s_ * (T[i] - 1));
          step[i] = static_cast<int>(-s_);
          if (!used(i)) { lower[i] = upper[i] = 0; }
        }
        if (empty) {
          if (A[0] && A[1] && A[2])
            return set_err(TIR_B200_ERR_UNSUPPORTED, "T2D: kernel smaller than stride");
          continue;
        }
        tb::SubProb& s = p.sub[ns];
        set_sub_identity(s);
        const int64_t M = g.n * static_cast<int64_t>(A[0]) * A[1] * A[2];
        s.m_count = static_cast<int32_t>(M);
        m_max = std::max(m_max, M);
        s.gx = A[2];
        s.gy = A[1];
        s.gz = A[0];
        for (int i = 0; i < 3; ++i) {
          s.a_lo[i] = lower[2 - i];
          s.a_st[i] = 1;
          s.taps[i] = T[2 - i];
          s.a_dil[i] = 1;
          s.w_base[i] = base[2 - i];
          s.w_step[i] = step[2 - i];
          s.o_st[i] = static_cast<int32_t>(g.s[2 - i]);
          s.o_b[i] = q[2 - i];
        }
        s.num_pieces = T[0] * T[1] * T[2] * p.cb_per_tap;
        int rc = encode_im2col(&p.tmA[ns], X, g, g.ci, rank, lower, upper, estr, box);
        if (rc) return rc;
        ++ns;
      }
  p.num_sub = ns;
  if (ns == 0) return set_err(TIR_B200_ERR_UNSUPPORTED, "T2D: no output classes");
  int kmax = 0;
  for (int i = 0; i < ns; ++i) kmax = std::max(kmax, p.sub[i].taps[0] * p.sub[i].taps[1] * p.sub[i].taps[2]);
  const int bn = choose_bn(cog, (m_max + tb::kBM - 1) / tb::kBM * ns, 1, kmax * ((cig + 15) / 16), di.sms,
                           !out_f16 && !epi.on());
  int max_pieces = 0;
  for (int i = 0; i < ns; ++i) max_pieces = std::max(max_pieces, p.sub[i].num_pieces);
  int ks = choose_ks(max_pieces, box, bn);
  if (bn >= 128) ks = std::min(ks, 2);
  int rc = encode_2d(&p.tmB, W, taps * cig, g.co, std::min(bn, 64), box);
  if (rc) return rc;
  p.ksplit = 1;
  rc = finalize_tiles(p, bn, ks);
  if (rc) return rc;
  p.ksplit = choose_ksplit(p, p.total_tiles, out_f16, di.sms);
  if (p.ksplit > 1) {
    rc = finalize_tiles(p, bn, ks);
    if (rc) return rc;
  }
  p.store_mode = 0;  // class rows scatter to strided output pixels
  return launch_igemm(p, bn, ks, stream);
}

// ------------------------------------------------------------------ DEP

// Tile shape per output width: 128 threads = 4 channel vectors x (TC/T) columns
// x (TR/R) rows; a narrow image (MobileNet-V2's 14x14 / 7x7 stages) gets a
// narrower tile so the footprint is not mostly padding.
template <int K, int S, int R, int T, int TR, int TC>
int launch_dep_tile(const Geo& g, const uint16_t* X, const uint16_t* W, const float* Yin, void* Y,
                    int accumulate, int out_f16, const Epi& epi, cudaStream_t stream) {
  constexpr int FR = (TR - 1) * S + K, FC = (TC - 1) * S + K;
  tb::DepTileParams p;
  std::memset(&p, 0, sizeof p);
  const Driver* drv = driver();
  if (!drv->tiled) return set_err(TIR_B200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.ci), static_cast<cuuint64_t>(g.in[2]),
                        static_cast<cuuint64_t>(g.in[1]), static_cast<cuuint64_t>(g.n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.ci * 2), static_cast<cuuint64_t>(g.ci * 2 * g.in[2]),
                           static_cast<cuuint64_t>(g.ci * 2 * g.in[2] * g.in[1])};
  cuuint32_t box[4] = {32, FC, FR, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = drv->tiled(&p.tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<uint16_t*>(X), dims,
                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(TIR_B200_ERR_CUDA, "DEP tensor map failed (%d)", (int)r);
  p.W = reinterpret_cast<const __half*>(W);
  p.Yin = Yin;
  p.Y = Y;
  p.n = static_cast<int32_t>(g.n);
  p.c = static_cast<int32_t>(g.ci);
  p.oh = static_cast<int32_t>(g.out[1]);
  p.ow = static_cast<int32_t>(g.out[2]);
  p.pad_h = static_cast<int32_t>(g.p[1]);
  p.pad_w = static_cast<int32_t>(g.p[2]);
  p.tiles_h = static_cast<int32_t>((g.out[1] + TR - 1) / TR);
  p.tiles_w = static_cast<int32_t>((g.out[2] + TC - 1) / TC);
  p.cblocks = static_cast<int32_t>((g.ci + 31) / 32);  // a partial last block when C % 32 != 0
  p.accumulate = accumulate;
  p.bias = epi.bias;
  p.relu = epi.relu;
  p.out_f16 = out_f16;
  p.trace = g_trace;
  const int64_t blocks = g.n * p.tiles_h * p.tiles_w * p.cblocks;
  if (blocks >= (1ll << 31)) return set_err(TIR_B200_ERR_UNSUPPORTED, "DEP: too many tiles");
  const size_t smem = 2 * ((static_cast<size_t>(FR) * FC * 32 * 2 + 127) / 128 * 128);  // two-slot ring
  // The epilogue is a template flag so the plain kernel keeps its register budget.
  auto kern = epi.on() ? tb::dep_tile_kernel<K, S, R, T, TR, TC, true>
                       : tb::dep_tile_kernel<K, S, R, T, TR, TC, false>;
  CUDA_TRY(ensure_smem(kern, smem));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
  const DeviceInfo di = device_info();
  const int grid = static_cast<int>(std::min<int64_t>(blocks, static_cast<int64_t>(std::max(per_sm, 1)) * di.sms));
  CUDA_TRY(launch_pdl(kern, grid, 128, smem, stream, p));
  ++g_launches;
  return TIR_B200_OK;
}

int dep_impl(const Geo& g, const uint16_t* X, const uint16_t* W, const float* Yin, void* Y,
             int accumulate, int out_f16, const Epi& epi, cudaStream_t stream) {
  if (g.in[0] != 1 || g.k[0] != 1)
    return set_err(TIR_B200_ERR_UNSUPPORTED, "DEP: 2-D (NHWC) depthwise only");
  if (epi.residual) return set_err(TIR_B200_ERR_UNSUPPORTED, "DEP: residual epilogue not supported");
  // Fast path: 3x3, stride 1 or 2, no dilation, 32-channel blocks, aligned operands.
  // fp32 outputs are written as 32-byte vectors (dep.cuh st.global.v8)
  const bool aligned = (reinterpret_cast<uintptr_t>(W) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(Y) % (out_f16 ? 16 : 32) == 0) &&
                       (!accumulate || reinterpret_cast<uintptr_t>(Yin) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(X) % 16 == 0);
  if (!tb::options().dep_simple && aligned && g.ci % 8 == 0 && g.ci >= 32 && g.k[1] == 3 && g.k[2] == 3 &&
      g.d[1] == 1 && g.d[2] == 1 && g.s[1] == g.s[2] && (g.s[1] == 1 || g.s[1] == 2)) {
    const int64_t ow = g.out[2];
    const int tc = tb::options().dep_tc;  // tile-width override (tuning)
    if (g.s[1] == 1 && tc == 16)
      return launch_dep_tile<3, 1, 4, 2, 16, 16>(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
    if (g.s[1] == 1 && tc == 8)
      return launch_dep_tile<3, 1, 1, 2, 8, 8>(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
    if (g.s[1] == 1) {
      // Tile shape (tools/sweep_options.py over the MobileNet-V2 shapes): the kernel is
      // issue-bound, so columns of a partial tile cost time — 16 x 16 when it divides the
      // width and 8 x 32 does not (112: 10.6 -> 10.2 us); narrow images take 8 x 8 tiles
      // while those fit in two waves of CTAs (14² C384: 5.4 -> 4.8 us), else 16 x 16.
      if (ow >= 24) {
        if (ow % 32 && ow % 16 == 0)
          return launch_dep_tile<3, 1, 4, 2, 16, 16>(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
        return launch_dep_tile<3, 1, 4, 2, 8, 32>(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
      }
      const int64_t tiles8 = g.n * ((g.out[1] + 7) / 8) * ((ow + 7) / 8) * ((g.ci + 31) / 32);
      if (ow >= 12 && tiles8 > 2 * 3 * static_cast<int64_t>(device_info().sms))
        return launch_dep_tile<3, 1, 4, 2, 16, 16>(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
      return launch_dep_tile<3, 1, 1, 2, 8, 8>(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
    }
    if (ow >= 12) return launch_dep_tile<3, 2, 2, 2, 8, 16>(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
    return launch_dep_tile<3, 2, 1, 2, 8, 8>(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
  }
  tb::DepParams p;
  p.X = reinterpret_cast<const __half*>(X);
  p.W = reinterpret_cast<const __half*>(W);
  p.Yin = Yin;
  p.Y = Y;
  p.n = static_cast<int32_t>(g.n);
  p.ih = static_cast<int32_t>(g.in[1]);
  p.iw = static_cast<int32_t>(g.in[2]);
  p.c = static_cast<int32_t>(g.ci);
  p.oh = static_cast<int32_t>(g.out[1]);
  p.ow = static_cast<int32_t>(g.out[2]);
  p.kh = static_cast<int32_t>(g.k[1]);
  p.kw = static_cast<int32_t>(g.k[2]);
  p.sh = static_cast<int32_t>(g.s[1]);
  p.sw = static_cast<int32_t>(g.s[2]);
  p.ph = static_cast<int32_t>(g.p[1]);
  p.pw = static_cast<int32_t>(g.p[2]);
  p.dh = static_cast<int32_t>(g.d[1]);
  p.dw = static_cast<int32_t>(g.d[2]);
  p.accumulate = accumulate;
  p.bias = epi.bias;
  p.relu = epi.relu;
  p.out_f16 = out_f16;
  const DeviceInfo di = device_info();
  constexpr int R = 4;
  const bool vec = (g.ci % 8 == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(W) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(Y) % 32 == 0);
  const int v = vec ? 8 : 1;
  const int64_t work = g.n * ((g.out[1] + R - 1) / R) * g.out[2] * (g.ci / v);
  if (work >= (1ll << 31)) return set_err(TIR_B200_ERR_UNSUPPORTED, "DEP: too many outputs");
  const int64_t blocks = std::min<int64_t>((work + 255) / 256, static_cast<int64_t>(di.sms) * 16);
  if (vec)
    tb::dep_kernel<8, R><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(p);
  else
    tb::dep_kernel<1, R><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(p);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return TIR_B200_OK;
}

int conv_impl(const tir_b200_conv_desc* desc, const uint16_t* X, const uint16_t* W,
              const float* Yin, void* Y, int accumulate, int out_f16, const Epi& epi, cudaStream_t stream) {
  Geo g{};
  int rc = make_geo(desc, &g);
  if (rc) return rc;
  if (!X || !W || !Y || (accumulate && !Yin)) return set_err(TIR_B200_ERR_VALUE, "conv: null operand");
  // Depthwise (CI/G == 1) is not a dense contraction: CUDA-core kernel.
  if (desc->op == TIR_B200_DEP || is_depthwise(g)) {
    if (!is_depthwise(g)) return set_err(TIR_B200_ERR_VALUE, "DEP requires groups == ci == co");
    return dep_impl(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
  }
  rc = conv_rowpack_impl(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
  if (rc != kNotEligible) return rc;
  rc = conv_halo_impl(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
  if (rc != kNotEligible) return rc;
  return conv_tc_impl(g, X, W, Yin, Y, accumulate, out_f16, epi, stream);
}

// ------------------------------------------------------------------ host-buffer paths

constexpr int kHostMaxChunks = 16;

struct HostCache {
  int dev = -1;
  cudaStream_t stream = nullptr;
  cudaStream_t side[3] = {nullptr, nullptr, nullptr};  // batch-chunk pipeline: H2D, conv, D2H streams
  cudaEvent_t ev[2 * kHostMaxChunks + 1] = {};          // weights / per-chunk H2D done / conv done
  void* dbuf = nullptr;
  size_t dbytes = 0;
  int* dflag = nullptr;
};
thread_local HostCache t_host;

int host_prepare(size_t bytes, char** base) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (t_host.dev != dev) {
    tir_b200_release_host_cache();
    CUDA_TRY(cudaStreamCreateWithFlags(&t_host.stream, cudaStreamNonBlocking));
    for (auto& st : t_host.side) CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto& e : t_host.ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&t_host.dflag), sizeof(int)));
    t_host.dev = dev;
  }
  if (t_host.dbytes < bytes) {
    if (t_host.dbuf) cudaFree(t_host.dbuf);
    t_host.dbuf = nullptr;
    t_host.dbytes = 0;
    CUDA_TRY(cudaMalloc(&t_host.dbuf, bytes));
    t_host.dbytes = bytes;
  }
  *base = static_cast<char*>(t_host.dbuf);
  return TIR_B200_OK;
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

// H2D of f32 host values, then device RN conversion to fp16 with an exactness flag.
int upload_f32_as_f16(const float* host, size_t n, float* dstage, uint16_t* d16, cudaStream_t st) {
  CUDA_TRY(cudaMemcpyAsync(dstage, host, n * 4, cudaMemcpyHostToDevice, st));
  if (tb::launch_f32_to_f16_exact(dstage, d16, static_cast<int64_t>(n), t_host.dflag, st))
    return set_err(TIR_B200_ERR_CUDA, "convert kernel launch failed");
  ++g_launches;
  return TIR_B200_OK;
}

}  // namespace

// ====================================================================== C-ABI

extern "C" {

int tir_b200_version(void) { return 1; }
void tir_b200_debug_set_trace(unsigned long long* dev_buf) { g_trace = dev_buf; }
const char* tir_b200_last_error(void) { return g_err.c_str(); }
int64_t tir_b200_launch_count(void) { return g_launches; }
void tir_b200_reset_launch_count(void) { g_launches = 0; }

int tir_b200_release_workspaces(void) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  int cur = 0;
  CUDA_TRY(cudaGetDevice(&cur));
  CUDA_TRY(cudaDeviceSynchronize());
  for (void* p : g_ws_retired) cudaFree(p);
  for (Workspace& w : g_ws) {
    cudaSetDevice(w.dev);
    cudaDeviceSynchronize();
    cudaFree(w.ptr);
  }
  cudaSetDevice(cur);
  g_ws_retired.clear();
  g_ws.clear();
  return TIR_B200_OK;
}

int tir_b200_set_option(const char* name, int value) {
  int n = 0;
  const tb::OptionEntry* t = tb::option_table(&n);
  for (int i = 0; name && i < n; ++i)
    if (!strcmp(name, t[i].name)) {
      tb::options().*(t[i].field) = value;
      return TIR_B200_OK;
    }
  return set_err(TIR_B200_ERR_VALUE, "unknown option '%s'", name ? name : "(null)");
}

int tir_b200_get_option(const char* name, int* value) {
  int n = 0;
  const tb::OptionEntry* t = tb::option_table(&n);
  for (int i = 0; name && value && i < n; ++i)
    if (!strcmp(name, t[i].name)) {
      *value = tb::options().*(t[i].field);
      return TIR_B200_OK;
    }
  return set_err(TIR_B200_ERR_VALUE, "unknown option '%s'", name ? name : "(null)");
}

int tir_b200_conv_out_shape(const tir_b200_conv_desc* desc, int64_t out_dhw[3]) {
  Geo g{};
  int rc = make_geo(desc, &g);
  if (rc) return rc;
  for (int i = 0; i < 3; ++i) out_dhw[i] = g.out[i];
  return TIR_B200_OK;
}

int tir_b200_gmm(const uint16_t* A, const uint16_t* B, const float* Cin, void* C, int64_t M,
                 int64_t N, int64_t K, int accumulate, int out_f16, void* stream) {
  return gmm_impl(A, B, Cin, C, M, N, K, accumulate, out_f16, Epi{}, static_cast<cudaStream_t>(stream));
}

int tir_b200_gmm_ex(const uint16_t* A, const uint16_t* B, const float* Cin, void* C, int64_t M,
                    int64_t N, int64_t K, int accumulate, int out_f16, const tir_b200_epilogue* epi,
                    void* stream) {
  return gmm_impl(A, B, Cin, C, M, N, K, accumulate, out_f16, make_epi(epi),
                  static_cast<cudaStream_t>(stream));
}

int tir_b200_conv(const tir_b200_conv_desc* desc, const uint16_t* X, const uint16_t* W,
                  const float* Yin, void* Y, int accumulate, int out_f16, void* stream) {
  return conv_impl(desc, X, W, Yin, Y, accumulate, out_f16, Epi{}, static_cast<cudaStream_t>(stream));
}

int tir_b200_conv_ex(const tir_b200_conv_desc* desc, const uint16_t* X, const uint16_t* W,
                     const float* Yin, void* Y, int accumulate, int out_f16,
                     const tir_b200_epilogue* epi, void* stream) {
  return conv_impl(desc, X, W, Yin, Y, accumulate, out_f16, make_epi(epi),
                   static_cast<cudaStream_t>(stream));
}

int tir_b200_gmm_host(const uint16_t* A, const uint16_t* B, float* C, int64_t M, int64_t N,
                      int64_t K, int accumulate) {
  if (M < 0 || N < 0 || K < 0) return set_err(TIR_B200_ERR_VALUE, "gmm: negative extent");
  const size_t a = align256(M * K * 2), b = align256(K * N * 2), c = align256(M * N * 4);
  char* d = nullptr;
  int rc = host_prepare(a + b + c, &d);
  if (rc) return rc;
  cudaStream_t st = t_host.stream;
  CUDA_TRY(cudaMemcpyAsync(d, A, M * K * 2, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d + a, B, K * N * 2, cudaMemcpyHostToDevice, st));
  if (accumulate) CUDA_TRY(cudaMemcpyAsync(d + a + b, C, M * N * 4, cudaMemcpyHostToDevice, st));
  rc = gmm_impl(reinterpret_cast<uint16_t*>(d), reinterpret_cast<uint16_t*>(d + a),
                reinterpret_cast<float*>(d + a + b), d + a + b, M, N, K, accumulate, 0, Epi{}, st);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(C, d + a + b, M * N * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TIR_B200_OK;
}

// debug (tools/e2e_probe.py): host microseconds of the last tir_b200_conv_host call —
// [0] until every chunk is enqueued, [1] until the final synchronize returned
static double g_host_times[2];
void tir_b200_debug_host_times(double* out) {
  out[0] = g_host_times[0];
  out[1] = g_host_times[1];
}
int tir_b200_conv_host(const tir_b200_conv_desc* desc, const uint16_t* X, const uint16_t* W,
                       float* Y, int accumulate) {
  const auto t_entry = std::chrono::steady_clock::now();
  Geo g{};
  int rc = make_geo(desc, &g);
  if (rc) return rc;
  const int64_t xe = g.n * g.in[0] * g.in[1] * g.in[2] * g.ci;
  const int64_t we = g.k[0] * g.k[1] * g.k[2] * (g.ci / g.g) * g.co;
  const int64_t ye = g.n * g.out[0] * g.out[1] * g.out[2] * g.co;
  const size_t xa = align256(xe * 2), wa = align256(we * 2), ya = align256(ye * 4);
  char* d = nullptr;
  rc = host_prepare(xa + wa + ya, &d);
  if (rc) return rc;
  cudaStream_t st = t_host.stream;
  CUDA_TRY(cudaMemcpyAsync(d + xa, W, we * 2, cudaMemcpyHostToDevice, st));
  // Batch-chunk pipeline: images are independent (every output keeps its own
  // reduction order, so a batch slice is bit-identical), so the chunks' H2D, conv
  // and D2H overlap. Only for convs that need no shared library workspace
  // (CI / G a multiple of 8: no relayout kernels).
  const int64_t cig = g.ci / g.g;
  const int nch = (cig % 8 == 0 && g.n >= 2 && tb::options().host_pipeline)
                      ? static_cast<int>(std::min<int64_t>(g.n, tb::options().host_chunks)) : 1;
  const int64_t x_img = xe / g.n, y_img = ye / g.n;
  const int nchunks = std::min(nch, kHostMaxChunks);
  // Three streams: the H2D copies back to back on one, the convs on another, the
  // D2H copies on a third (each waiting on its chunk's event), so the two copy
  // directions and the GPU overlap across chunks without a chunk's D2H delaying
  // a later chunk's H2D on a shared stream.
  cudaStream_t sh = t_host.side[0], sc = t_host.side[1], sd = t_host.side[2];
  CUDA_TRY(cudaEventRecord(t_host.ev[0], st));  // weights uploaded
  CUDA_TRY(cudaStreamWaitEvent(sc, t_host.ev[0], 0));
  CUDA_TRY(cudaStreamWaitEvent(sh, t_host.ev[0], 0));  // buffers free of the previous call's work on st
  for (int c = 0; c < nchunks; ++c) {
    const int64_t n0 = g.n * c / nchunks, n1 = g.n * (c + 1) / nchunks;
    uint16_t* dx = reinterpret_cast<uint16_t*>(d) + n0 * x_img;
    float* dy = reinterpret_cast<float*>(d + xa + wa) + n0 * y_img;
    CUDA_TRY(cudaMemcpyAsync(dx, X + n0 * x_img, (n1 - n0) * x_img * 2, cudaMemcpyHostToDevice, sh));
    if (accumulate) CUDA_TRY(cudaMemcpyAsync(dy, Y + n0 * y_img, (n1 - n0) * y_img * 4, cudaMemcpyHostToDevice, sh));
    CUDA_TRY(cudaEventRecord(t_host.ev[1 + c], sh));
    CUDA_TRY(cudaStreamWaitEvent(sc, t_host.ev[1 + c], 0));
    tir_b200_conv_desc dc = *desc;
    dc.n = n1 - n0;
    rc = conv_impl(&dc, dx, reinterpret_cast<uint16_t*>(d + xa), dy, dy, accumulate, 0, Epi{}, sc);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(t_host.ev[1 + kHostMaxChunks + c], sc));
    CUDA_TRY(cudaStreamWaitEvent(sd, t_host.ev[1 + kHostMaxChunks + c], 0));
    CUDA_TRY(cudaMemcpyAsync(Y + n0 * y_img, dy, (n1 - n0) * y_img * 4, cudaMemcpyDeviceToHost, sd));
  }
  const auto t_enq = std::chrono::steady_clock::now();
  CUDA_TRY(cudaStreamSynchronize(sd));
  const auto t_end = std::chrono::steady_clock::now();
  g_host_times[0] = std::chrono::duration<double, std::micro>(t_enq - t_entry).count();
  g_host_times[1] = std::chrono::duration<double, std::micro>(t_end - t_entry).count();
  return TIR_B200_OK;
}

static int check_exact_flag() {
  int flag = 0;
  CUDA_TRY(cudaMemcpyAsync(&flag, t_host.dflag, sizeof(int), cudaMemcpyDeviceToHost, t_host.stream));
  CUDA_TRY(cudaStreamSynchronize(t_host.stream));
  if (flag) return set_err(TIR_B200_ERR_VALUE, "inexact f16 input: a value is not representable in fp16");
  return TIR_B200_OK;
}

int tir_b200_gmm_host_f32(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                          int accumulate) {
  if (M < 0 || N < 0 || K < 0) return set_err(TIR_B200_ERR_VALUE, "gmm: negative extent");
  const size_t a = align256(M * K * 2), b = align256(K * N * 2), c = align256(M * N * 4);
  const size_t stage = align256(std::max(M * K, K * N) * 4);
  char* d = nullptr;
  int rc = host_prepare(a + b + c + stage, &d);
  if (rc) return rc;
  cudaStream_t st = t_host.stream;
  CUDA_TRY(cudaMemsetAsync(t_host.dflag, 0, sizeof(int), st));
  float* sg = reinterpret_cast<float*>(d + a + b + c);
  rc = upload_f32_as_f16(A, M * K, sg, reinterpret_cast<uint16_t*>(d), st);
  if (rc) return rc;
  rc = upload_f32_as_f16(B, K * N, sg, reinterpret_cast<uint16_t*>(d + a), st);
  if (rc) return rc;
  rc = check_exact_flag();
  if (rc) return rc;
  if (accumulate) CUDA_TRY(cudaMemcpyAsync(d + a + b, C, M * N * 4, cudaMemcpyHostToDevice, st));
  rc = gmm_impl(reinterpret_cast<uint16_t*>(d), reinterpret_cast<uint16_t*>(d + a),
                reinterpret_cast<float*>(d + a + b), d + a + b, M, N, K, accumulate, 0, Epi{}, st);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(C, d + a + b, M * N * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TIR_B200_OK;
}

int tir_b200_conv_host_f32(const tir_b200_conv_desc* desc, const float* X, const float* W, float* Y,
                           int accumulate) {
  Geo g{};
  int rc = make_geo(desc, &g);
  if (rc) return rc;
  const int64_t xe = g.n * g.in[0] * g.in[1] * g.in[2] * g.ci;
  const int64_t we = g.k[0] * g.k[1] * g.k[2] * (g.ci / g.g) * g.co;
  const int64_t ye = g.n * g.out[0] * g.out[1] * g.out[2] * g.co;
  const size_t xa = align256(xe * 2), wa = align256(we * 2), ya = align256(ye * 4);
  const size_t stage = align256(std::max(xe, we) * 4);
  char* d = nullptr;
  rc = host_prepare(xa + wa + ya + stage, &d);
  if (rc) return rc;
  cudaStream_t st = t_host.stream;
  CUDA_TRY(cudaMemsetAsync(t_host.dflag, 0, sizeof(int), st));
  float* sg = reinterpret_cast<float*>(d + xa + wa + ya);
  rc = upload_f32_as_f16(X, xe, sg, reinterpret_cast<uint16_t*>(d), st);
  if (rc) return rc;
  rc = upload_f32_as_f16(W, we, sg, reinterpret_cast<uint16_t*>(d + xa), st);
  if (rc) return rc;
  rc = check_exact_flag();
  if (rc) return rc;
  if (accumulate) CUDA_TRY(cudaMemcpyAsync(d + xa + wa, Y, ye * 4, cudaMemcpyHostToDevice, st));
  rc = conv_impl(desc, reinterpret_cast<uint16_t*>(d), reinterpret_cast<uint16_t*>(d + xa),
                 reinterpret_cast<float*>(d + xa + wa), d + xa + wa, accumulate, 0, Epi{}, st);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(Y, d + xa + wa, ye * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TIR_B200_OK;
}

// ---- network-graph glue

static int check_vec(const void* a, const void* b, int64_t c) {
  if (!a || !b) return set_err(TIR_B200_ERR_VALUE, "null operand");
  if ((reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(b) & 15))
    return set_err(TIR_B200_ERR_UNSUPPORTED, "operands must be 16-byte aligned");
  if (c <= 0 || c % 8) return set_err(TIR_B200_ERR_UNSUPPORTED, "channels/cols must be a positive multiple of 8");
  return TIR_B200_OK;
}

int tir_b200_maxpool2d(const uint16_t* X, uint16_t* Y, int64_t n, int64_t h, int64_t w, int64_t c,
                       int64_t k, int64_t s, int64_t p, void* stream) {
  int rc = check_vec(X, Y, c);
  if (rc) return rc;
  if (n < 0 || h <= 0 || w <= 0 || k <= 0 || s <= 0 || p < 0 || p >= k)
    return set_err(TIR_B200_ERR_VALUE, "maxpool2d: bad geometry");
  const int64_t oh = (h + 2 * p - k) / s + 1, ow = (w + 2 * p - k) / s + 1;
  if (oh <= 0 || ow <= 0) return set_err(TIR_B200_ERR_VALUE, "maxpool2d: empty output");
  const int64_t total = n * oh * ow * (c / 8);
  if (total == 0) return TIR_B200_OK;
  const DeviceInfo di = device_info();
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, di.sms * 16));
  tb::maxpool2d_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      X, Y, (int)n, (int)h, (int)w, (int)c, (int)oh, (int)ow, (int)k, (int)s, (int)p);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return TIR_B200_OK;
}

int tir_b200_avgpool_global(const uint16_t* X, uint16_t* Y, int64_t n, int64_t hw, int64_t c, void* stream) {
  int rc = check_vec(X, Y, c);
  if (rc) return rc;
  if (n < 0 || hw <= 0 || n > 65535) return set_err(TIR_B200_ERR_VALUE, "avgpool_global: bad geometry");
  if (n == 0) return TIR_B200_OK;
  const int cv = static_cast<int>(c / 8);
  dim3 grid((cv + 63) / 64, static_cast<unsigned>(n));
  tb::avgpool_global_kernel<<<grid, 64, 0, static_cast<cudaStream_t>(stream)>>>(X, Y, (int)hw, (int)c);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return TIR_B200_OK;
}

int tir_b200_layernorm(const uint16_t* X, uint16_t* Y, const float* gamma, const float* beta, int64_t rows,
                       int64_t cols, float eps, void* stream) {
  int rc = check_vec(X, Y, cols);
  if (rc) return rc;
  if (!gamma || !beta) return set_err(TIR_B200_ERR_VALUE, "layernorm: null gamma/beta");
  if (cols > 8192 || rows < 0 || rows >= (1ll << 31)) return set_err(TIR_B200_ERR_UNSUPPORTED, "layernorm: shape");
  if (rows == 0) return TIR_B200_OK;
  const int cv = static_cast<int>(cols / 8);
  auto st = static_cast<cudaStream_t>(stream);
  if ((reinterpret_cast<uintptr_t>(gamma) & 15) == 0 && (reinterpret_cast<uintptr_t>(beta) & 15) == 0 &&
      cv <= 256) {  // warp per row
    const unsigned gw = static_cast<unsigned>((rows + 7) / 8);
    if (cv <= 32) tb::layernorm_warp_kernel<1><<<gw, 256, 0, st>>>(X, Y, gamma, beta, (int)rows, (int)cols, eps);
    else if (cv <= 64) tb::layernorm_warp_kernel<2><<<gw, 256, 0, st>>>(X, Y, gamma, beta, (int)rows, (int)cols, eps);
    else if (cv <= 128) tb::layernorm_warp_kernel<4><<<gw, 256, 0, st>>>(X, Y, gamma, beta, (int)rows, (int)cols, eps);
    else tb::layernorm_warp_kernel<8><<<gw, 256, 0, st>>>(X, Y, gamma, beta, (int)rows, (int)cols, eps);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    return TIR_B200_OK;
  }
  const int threads = std::min(256, (cv + 31) / 32 * 32);
  const int vpt = (cv + threads - 1) / threads;
  const unsigned g = static_cast<unsigned>(rows);
  if (vpt == 1) tb::layernorm_kernel<1><<<g, threads, 0, st>>>(X, Y, gamma, beta, (int)cols, eps);
  else if (vpt == 2) tb::layernorm_kernel<2><<<g, threads, 0, st>>>(X, Y, gamma, beta, (int)cols, eps);
  else tb::layernorm_kernel<4><<<g, threads, 0, st>>>(X, Y, gamma, beta, (int)cols, eps);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return TIR_B200_OK;
}

int tir_b200_softmax(const uint16_t* X, uint16_t* Y, int64_t rows, int64_t cols, float scale, void* stream) {
  int rc = check_vec(X, Y, cols);
  if (rc) return rc;
  if (cols > 8192 || rows < 0 || rows >= (1ll << 31)) return set_err(TIR_B200_ERR_UNSUPPORTED, "softmax: shape");
  if (rows == 0) return TIR_B200_OK;
  const int cv = static_cast<int>(cols / 8);
  auto st = static_cast<cudaStream_t>(stream);
  if (cv <= 256) {  // warp per row
    const unsigned gw = static_cast<unsigned>((rows + 7) / 8);
    if (cv <= 32) tb::softmax_warp_kernel<1><<<gw, 256, 0, st>>>(X, Y, (int)rows, (int)cols, scale);
    else if (cv <= 64) tb::softmax_warp_kernel<2><<<gw, 256, 0, st>>>(X, Y, (int)rows, (int)cols, scale);
    else if (cv <= 128) tb::softmax_warp_kernel<4><<<gw, 256, 0, st>>>(X, Y, (int)rows, (int)cols, scale);
    else tb::softmax_warp_kernel<8><<<gw, 256, 0, st>>>(X, Y, (int)rows, (int)cols, scale);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    return TIR_B200_OK;
  }
  const int threads = std::min(256, (cv + 31) / 32 * 32);
  const int vpt = (cv + threads - 1) / threads;
  const unsigned g = static_cast<unsigned>(rows);
  if (vpt == 1) tb::softmax_kernel<1><<<g, threads, 0, st>>>(X, Y, (int)cols, scale);
  else if (vpt == 2) tb::softmax_kernel<2><<<g, threads, 0, st>>>(X, Y, (int)cols, scale);
  else tb::softmax_kernel<4><<<g, threads, 0, st>>>(X, Y, (int)cols, scale);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return TIR_B200_OK;
}

int tir_b200_gmm_batched(const uint16_t* A, int64_t a_rows, int64_t lda, const uint16_t* B, int64_t b_rows,
                         int64_t ldb, void* C, int64_t c_rows, int64_t ldc, int64_t M, int64_t N, int64_t K,
                         const tir_b200_batch_desc* batch, int out_f16, const tir_b200_epilogue* epi,
                         void* stream) {
  return gmm_batched_impl(A, a_rows, lda, B, b_rows, ldb, C, c_rows, ldc, M, N, K, batch, out_f16,
                          make_epi(epi), static_cast<cudaStream_t>(stream));
}

void tir_b200_release_host_cache(void) {
  if (t_host.dev >= 0) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(t_host.dev);
    if (t_host.dbuf) cudaFree(t_host.dbuf);
    if (t_host.dflag) cudaFree(t_host.dflag);
    if (t_host.stream) cudaStreamDestroy(t_host.stream);
    for (auto st : t_host.side)
      if (st) cudaStreamDestroy(st);
    for (auto e : t_host.ev)
      if (e) cudaEventDestroy(e);
    cudaSetDevice(cur);
  }
  t_host = HostCache{};
}

}  // extern "C"
