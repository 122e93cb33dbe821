// prep.cuh — bit-exact layout / conversion steps around the contraction kernel.
//
//  * pad_channels: X[..., C] -> Xp[..., Cp] with zero channels (Cp = C rounded up
//    to 8). TMA needs a 16-byte pixel pitch; the CI = 3 first layers (C3D, DIL,
//    SURVEY §7 "hard parts") go through this. Zero channels meet zero weight
//    rows, so every real product and partial sum is unchanged.
//  * pad_weight_rows: W[taps, C, CO] -> Wp[taps, Cp, CO], zero rows.
//  * f32_to_f16_exact: the host-buffer entry points receive the interpreter's
//    f32 storage of F16 values (ir.cc:36-47); convert with RN and flag any
//    value that does not survive the round trip (rejected as ValueError).
#pragma once

#include <algorithm>

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "options.h"

namespace tb {

__global__ void pad_channels_kernel(const uint16_t* __restrict__ x, uint16_t* __restrict__ y,
                                    int64_t pixels, int32_t c, int32_t cp) {
  const int64_t total = pixels * cp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pix = i / cp;
    const int32_t ch = static_cast<int32_t>(i - pix * cp);
    y[i] = ch < c ? x[pix * c + ch] : static_cast<uint16_t>(0);
  }
}

__global__ void pad_weight_rows_kernel(const uint16_t* __restrict__ w, uint16_t* __restrict__ y,
                                       int64_t taps, int32_t c, int32_t cp, int32_t co) {
  const int64_t total = taps * cp * co;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t col = i % co;
    const int64_t row = i / co;
    const int64_t tap = row / cp;
    const int32_t ch = static_cast<int32_t>(row - tap * cp);
    y[i] = ch < c ? w[(tap * c + ch) * co + col] : static_cast<uint16_t>(0);
  }
}

__global__ void f32_to_f16_exact_kernel(const float* __restrict__ x, uint16_t* __restrict__ y,
                                        int64_t n, int* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = x[i];
    const __half h = __float2half_rn(v);
    const float back = __half2float(h);
    // NaN never compares equal; the reference's f16 tag stores finite values.
    if (!(back == v)) bad = true;
    y[i] = __half_as_ushort(h);
  }
  if (bad) atomicExch(flag, 1);
}

// (kw, c) packing for small-channel convs (the CI = 3 first layers, C3D/DIL):
//   Xp[n, d, h, ow, t*C + c] = X[n, d, h, ow*sw - pw + t*dw, c]   (0 if out of bounds)
//   Wp[(kd, kh), t*C + c, co] = W[(kd, kh, t), c, co]             (zero rows past KW*C)
// so the convolution becomes a (KD, KH, 1) convolution over Xp with Cp = KW*C
// rounded up to 8/16/32 channels: a pure relayout (zero fill = the reference's
// select(in-bounds, x, 0.0) padding), so every product and partial sum is the same.
__global__ void pack_kw_kernel(const uint16_t* __restrict__ x, uint16_t* __restrict__ y, int64_t rows,
                               int32_t iw, int32_t c, int32_t ow, int32_t kw, int32_t sw, int32_t pw,
                               int32_t dw, int32_t cp) {
  // one thread per (row, ow, 8-channel group); row = n*D*H flattened
  const int groups = cp / 8;
  const int64_t total = rows * ow * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int grp = static_cast<int>(i % groups);
    const int64_t pix = i / groups;  // row * ow + o
    const int o = static_cast<int>(pix % ow);
    const int64_t row = pix / ow;
    const uint16_t* xr = x + row * iw * c;
    uint16_t v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = grp * 8 + e;
      const int t = j / c, ch = j - t * c;
      const int wi = o * sw - pw + t * dw;
      v[e] = (t < kw && wi >= 0 && wi < iw) ? xr[wi * c + ch] : static_cast<uint16_t>(0);
    }
    uint4 u;
    u.x = v[0] | (static_cast<uint32_t>(v[1]) << 16);
    u.y = v[2] | (static_cast<uint32_t>(v[3]) << 16);
    u.z = v[4] | (static_cast<uint32_t>(v[5]) << 16);
    u.w = v[6] | (static_cast<uint32_t>(v[7]) << 16);
    *reinterpret_cast<uint4*>(y + pix * cp + grp * 8) = u;
  }
}

__global__ void pack_kw_weights_kernel(const uint16_t* __restrict__ w, uint16_t* __restrict__ y,
                                       int64_t khd, int32_t kwc, int32_t cp, int32_t co) {
  const int64_t total = khd * cp * co;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t col = i % co;
    const int64_t row = i / co;
    const int64_t g = row / cp;
    const int32_t j = static_cast<int32_t>(row - g * cp);
    y[i] = j < kwc ? w[(g * kwc + j) * co + col] : static_cast<uint16_t>(0);
  }
}

// (kw, c) packing of X and of the weights in ONE launch (replaces the two
// kernels above on the hot path). Blocks [0, rows) each relayout one input row
// (n, d, h): the row (iw * c halves, <= 48 KB) is staged in shared memory with
// 16-byte loads, then every 16-byte output vector (o, 8 packed channels) is
// gathered from it; per-row indices stay 32-bit and the (t, ch) split of a
// packed channel comes from a small table (the old per-element int64 div/mod
// made the relayout run at 1.5 TB/s). Blocks [rows, rows + wblocks) pack the
// weights [khd][kwc][co] -> [khd][cp][co] (zero rows j >= kwc).
__global__ void __launch_bounds__(256) pack_kw_fused_kernel(
    const uint16_t* __restrict__ x, uint16_t* __restrict__ y, const uint16_t* __restrict__ w,
    uint16_t* __restrict__ wy, int32_t rows, int32_t rpb, int32_t xblocks, int32_t iw, int32_t c, int32_t ow,
    int32_t kw, int32_t sw, int32_t pw, int32_t dw, int32_t cp, int32_t khd, int32_t kwc, int32_t co) {
  extern __shared__ __align__(16) uint16_t srow[];  // rpb staged input rows
  __shared__ int16_t tab_t[64], tab_c[64];
  if (static_cast<int32_t>(blockIdx.x) >= xblocks) {  // weights
    const int64_t total = static_cast<int64_t>(khd) * cp * co;
    const int64_t step = static_cast<int64_t>(gridDim.x - xblocks) * blockDim.x;
    for (int64_t i = (blockIdx.x - xblocks) * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += step) {
      const int32_t col = static_cast<int32_t>(i % co);
      const int64_t r = i / co;
      const int32_t g = static_cast<int32_t>(r / cp), j = static_cast<int32_t>(r % cp);
      wy[i] = j < kwc ? w[(static_cast<int64_t>(g) * kwc + j) * co + col] : static_cast<uint16_t>(0);
    }
    return;
  }
  if (threadIdx.x < cp) {
    tab_t[threadIdx.x] = static_cast<int16_t>(threadIdx.x / c);
    tab_c[threadIdx.x] = static_cast<int16_t>(threadIdx.x % c);
  }
  const int32_t row0 = blockIdx.x * rpb;
  const int32_t nrows = min(rpb, rows - row0);
  const int32_t row_elems = iw * c;
  const uint16_t* xr = x + static_cast<int64_t>(row0) * row_elems;
  // all rows of the block in flight at once (the loads are the latency-bound half)
  if ((row_elems & 7) == 0 && (reinterpret_cast<uintptr_t>(xr) & 15) == 0) {
    for (int v = threadIdx.x; v < nrows * row_elems / 8; v += blockDim.x)
      reinterpret_cast<uint4*>(srow)[v] = __ldg(reinterpret_cast<const uint4*>(xr) + v);
  } else {
    for (int v = threadIdx.x; v < nrows * row_elems; v += blockDim.x) srow[v] = __ldg(xr + v);
  }
  __syncthreads();
  const int32_t gshift = cp == 8 ? 0 : cp == 16 ? 1 : cp == 32 ? 2 : 3;  // log2(cp / 8)
  const int32_t nvec = ow << gshift;
  uint4* yb = reinterpret_cast<uint4*>(y + static_cast<int64_t>(row0) * ow * cp);
  for (int32_t v = threadIdx.x; v < nrows * nvec; v += blockDim.x) {
    const int32_t r = v / nvec, vr = v - r * nvec;
    const int32_t o = vr >> gshift, grp = vr & ((1 << gshift) - 1);
    const int32_t base = o * sw - pw;
    const uint16_t* sr = srow + r * row_elems;
    uint16_t e8[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int32_t j = grp * 8 + e;
      const int32_t t = tab_t[j], ch = tab_c[j];
      const int32_t wi = base + t * dw;
      e8[e] = (t < kw && wi >= 0 && wi < iw) ? sr[wi * c + ch] : static_cast<uint16_t>(0);
    }
    uint4 u;
    u.x = e8[0] | (static_cast<uint32_t>(e8[1]) << 16);
    u.y = e8[2] | (static_cast<uint32_t>(e8[3]) << 16);
    u.z = e8[4] | (static_cast<uint32_t>(e8[5]) << 16);
    u.w = e8[6] | (static_cast<uint32_t>(e8[7]) << 16);
    yb[v] = u;
  }
}

// Window form of the (kw, c) packing, for sw % dw == 0 (every stride-1 conv, and
// DIL / C3D's strided stems): stage S[q] = X[row, q*dw - pw, 0:c] (zero out of
// bounds) per input row; then output pixel o's packed vector is the CONTIGUOUS
// run S[o*(sw/dw) .. +kw) of kwc halves, followed by cp - kwc zeros. Each thread
// emits one 16-byte output vector from five aligned 32-bit shared loads and a
// funnel shift (no per-element gathers or index tables: the gather form spent
// ~24 shared loads per vector and ran the relayout at ~2.9 TB/s).
__global__ void __launch_bounds__(256) pack_kw_win_kernel(
    const uint16_t* __restrict__ x, uint16_t* __restrict__ y, const uint16_t* __restrict__ w,
    uint16_t* __restrict__ wy, int32_t rows, int32_t rpb, int32_t xblocks, int32_t iw, int32_t c, int32_t ow,
    int32_t sw_dw, int32_t pw, int32_t dw, int32_t slen, int32_t nstage, int32_t gshift, int32_t khd,
    int32_t kwc, int32_t co) {
  extern __shared__ __align__(16) uint16_t sst[];  // rpb rows of slen halves
  const int32_t cp = 8 << gshift;
  if (static_cast<int32_t>(blockIdx.x) >= xblocks) {  // weights
    const int64_t total = static_cast<int64_t>(khd) * cp * co;
    const int64_t step = static_cast<int64_t>(gridDim.x - xblocks) * blockDim.x;
    for (int64_t i = (blockIdx.x - xblocks) * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += step) {
      const int32_t col = static_cast<int32_t>(i % co);
      const int64_t r = i / co;
      const int32_t g = static_cast<int32_t>(r / cp), j = static_cast<int32_t>(r % cp);
      wy[i] = j < kwc ? w[(static_cast<int64_t>(g) * kwc + j) * co + col] : static_cast<uint16_t>(0);
    }
    return;
  }
  const int32_t row0 = blockIdx.x * rpb;
  const int32_t nrows = min(rpb, rows - row0);
  const int32_t row_elems = iw * c;
  const uint16_t* xr = x + static_cast<int64_t>(row0) * row_elems;
  // stage: nstage = (ow-1)*(sw/dw)*c + kw*c halves carry data, the rest of slen is zero
  for (int32_t i = threadIdx.x; i < nrows * slen; i += blockDim.x) {
    const int32_t r = i / slen, k = i - r * slen;
    uint16_t v = 0;
    if (k < nstage) {
      const int32_t q = k / c, ch = k - q * c;
      const int32_t col = q * dw - pw;
      if (col >= 0 && col < iw) v = __ldg(xr + r * row_elems + col * c + ch);
    }
    sst[i] = v;
  }
  __syncthreads();
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(sst);
  const int32_t nvec = ow << gshift;
  uint4* yb = reinterpret_cast<uint4*>(y + static_cast<int64_t>(row0) * ow * cp);
  for (int32_t v = threadIdx.x; v < nrows * nvec; v += blockDim.x) {
    const int32_t r = v / nvec, vr = v - r * nvec;
    const int32_t o = vr >> gshift, j0 = (vr & ((1 << gshift) - 1)) * 8;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (j0 < kwc) {
      const int32_t s = r * slen + o * sw_dw * c + j0;  // halves; slen is even
      const uint32_t* p = s32 + (s >> 1);
      uint32_t a[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) a[i] = p[i];
      uint32_t o4[4];
      const uint32_t sh = (s & 1) * 16;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t word = __funnelshift_r(a[i], a[i + 1], sh);
        const int32_t jl = j0 + 2 * i;
        if (jl >= kwc) word = 0;
        else if (jl + 1 >= kwc) word &= 0xffffu;
        o4[i] = word;
      }
      u = make_uint4(o4[0], o4[1], o4[2], o4[3]);
    }
    yb[v] = u;
  }
}

inline int launch_pack_kw_win(const uint16_t* x, uint16_t* y, const uint16_t* w, uint16_t* wy, int64_t rows,
                              int64_t iw, int64_t c, int64_t ow, int64_t kw, int64_t sw, int64_t pw, int64_t dw,
                              int64_t cp, int64_t khd, int64_t kwc, int64_t co, cudaStream_t st) {
  if (dw < 1 || sw % dw != 0 || cp > 64 || cp < 8 || rows >= (1ll << 30)) return 2;
  const int64_t sw_dw = sw / dw;
  const int64_t nstage = ((ow - 1) * sw_dw + kw) * c;
  // reads reach 8*ceil(kwc/8) + 2 halves past a window start
  const int64_t slen = ((ow - 1) * sw_dw * c + (kwc + 7) / 8 * 8 + 2 + 7) / 8 * 8;
  if (slen * 2 > 24 * 1024) return 2;
  const int rpb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, 12 * 1024 / (slen * 2))));
  const int64_t xblocks = (rows + rpb - 1) / rpb;
  const int wblocks = 16;
  const int gshift = cp == 8 ? 0 : cp == 16 ? 1 : cp == 32 ? 2 : 3;
  const size_t smem = static_cast<size_t>(rpb * slen * 2);
  pack_kw_win_kernel<<<static_cast<unsigned>(xblocks + wblocks), 256, smem, st>>>(
      x, y, w, wy, static_cast<int32_t>(rows), rpb, static_cast<int32_t>(xblocks), static_cast<int32_t>(iw),
      static_cast<int32_t>(c), static_cast<int32_t>(ow), static_cast<int32_t>(sw_dw), static_cast<int32_t>(pw),
      static_cast<int32_t>(dw), static_cast<int32_t>(slen), static_cast<int32_t>(nstage), gshift,
      static_cast<int32_t>(khd), static_cast<int32_t>(kwc), static_cast<int32_t>(co));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

inline int launch_pack_kw_fused(const uint16_t* x, uint16_t* y, const uint16_t* w, uint16_t* wy, int64_t rows,
                                int64_t iw, int64_t c, int64_t ow, int64_t kw, int64_t sw, int64_t pw, int64_t dw,
                                int64_t cp, int64_t khd, int64_t kwc, int64_t co, cudaStream_t st) {
  // Window form only for dilated strips (DIL: ~1 us faster); for dw = 1 (MobileNet /
  // C3D stems) the gather form's 16-byte staging loads win (MobileNet-V2 +1.5 %).
  if (dw > 1 && !options().pack_gather) {
    const int rc = launch_pack_kw_win(x, y, w, wy, rows, iw, c, ow, kw, sw, pw, dw, cp, khd, kwc, co, st);
    if (rc != 2) return rc;
  }
  const int64_t row_bytes = iw * c * 2;
  if (row_bytes > 48 * 1024 || rows >= (1ll << 30) || cp > 64) return 2;  // caller falls back
  const int rpb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, 12 * 1024 / row_bytes)));
  const int64_t xblocks = (rows + rpb - 1) / rpb;
  const int wblocks = 16;
  const size_t smem = static_cast<size_t>(rpb * row_bytes + 16);
  pack_kw_fused_kernel<<<static_cast<unsigned>(xblocks + wblocks), 256, smem, st>>>(
      x, y, w, wy, static_cast<int32_t>(rows), rpb, static_cast<int32_t>(xblocks), static_cast<int32_t>(iw),
      static_cast<int32_t>(c), static_cast<int32_t>(ow), static_cast<int32_t>(kw), static_cast<int32_t>(sw),
      static_cast<int32_t>(pw), static_cast<int32_t>(dw), static_cast<int32_t>(cp), static_cast<int32_t>(khd),
      static_cast<int32_t>(kwc), static_cast<int32_t>(co));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// (kh, kw, c) packing for CI = 3 stems whose KH*KW*CI exceeds 64 (C3D's and
// DIL's 7x7 windows, 147 values): Xp[n, d, oh, ow, j] = X[n, d, oh*sh - ph + kh*dh,
// ow*sw - pw + kw*dw, c] with j = (kh*KW + kw)*C + c (zero where out of bounds or
// j >= KH*KW*C), cp a multiple of 64 so the conv that remains (depth taps only)
// streams 64-channel im2col pieces instead of request-bound 32-channel ones.
// Block = one output row (n, d, oh): the KH input rows it needs (KH * W * C
// halves) are staged in shared memory; threads emit 16-byte output vectors from
// a (kh, kw, c) table. The weights [KD][KH][KW][C][CO] are already in j order
// per kd: Wp[kd][j][co] is a copy with zero rows j >= KH*KW*C (extra blocks).
__global__ void __launch_bounds__(256) pack_hw_kernel(
    const uint16_t* __restrict__ x, uint16_t* __restrict__ y, const uint16_t* __restrict__ w,
    uint16_t* __restrict__ wy, int32_t rows, int32_t ih, int32_t iw, int32_t c, int32_t oh, int32_t ow,
    int32_t kh, int32_t kw, int32_t sh, int32_t sw, int32_t ph, int32_t pw, int32_t dh, int32_t dw, int32_t cp,
    int32_t kd, int32_t co) {
  extern __shared__ __align__(16) uint16_t srows[];  // [kh][iw * c]
  __shared__ int16_t tab_h[256], tab_w[256], tab_c[256];
  const int32_t taps_c = kh * kw * c;
  if (static_cast<int32_t>(blockIdx.x) >= rows) {  // weights
    const int64_t total = static_cast<int64_t>(kd) * cp * co;
    const int64_t step = static_cast<int64_t>(gridDim.x - rows) * blockDim.x;
    for (int64_t i = (blockIdx.x - rows) * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += step) {
      const int32_t col = static_cast<int32_t>(i % co);
      const int64_t r = i / co;
      const int32_t g = static_cast<int32_t>(r / cp), j = static_cast<int32_t>(r % cp);
      wy[i] = j < taps_c ? w[(static_cast<int64_t>(g) * taps_c + j) * co + col] : static_cast<uint16_t>(0);
    }
    return;
  }
  for (int j = threadIdx.x; j < cp; j += blockDim.x) {
    const int t = j / c;
    tab_h[j] = static_cast<int16_t>(j < taps_c ? t / kw : -1);
    tab_w[j] = static_cast<int16_t>(t % kw);
    tab_c[j] = static_cast<int16_t>(j % c);
  }
  // row = (n*D + d)*OH + oy
  const int32_t oy = static_cast<int32_t>(blockIdx.x) % oh;
  const int64_t nd = static_cast<int64_t>(blockIdx.x) / oh;
  const int32_t row_elems = iw * c;
  for (int t = 0; t < kh; ++t) {
    const int32_t y_in = oy * sh - ph + t * dh;
    uint16_t* dst = srows + t * row_elems;
    if (y_in < 0 || y_in >= ih) {
      for (int v = threadIdx.x; v < row_elems; v += blockDim.x) dst[v] = 0;
    } else {
      const uint16_t* src = x + (nd * ih + y_in) * row_elems;
      for (int v = threadIdx.x; v < row_elems; v += blockDim.x) dst[v] = __ldg(src + v);
    }
  }
  __syncthreads();
  const int32_t nvec = ow * (cp / 8);
  uint4* yr = reinterpret_cast<uint4*>(y + static_cast<int64_t>(blockIdx.x) * ow * cp);
  for (int32_t v = threadIdx.x; v < nvec; v += blockDim.x) {
    const int32_t o = v / (cp / 8), grp = v - o * (cp / 8);
    const int32_t base = o * sw - pw;
    uint16_t e8[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int32_t j = grp * 8 + e;
      const int32_t th = tab_h[j];
      const int32_t wi = base + tab_w[j] * dw;
      e8[e] = (th >= 0 && wi >= 0 && wi < iw) ? srows[th * row_elems + wi * c + tab_c[j]] : static_cast<uint16_t>(0);
    }
    uint4 u;
    u.x = e8[0] | (static_cast<uint32_t>(e8[1]) << 16);
    u.y = e8[2] | (static_cast<uint32_t>(e8[3]) << 16);
    u.z = e8[4] | (static_cast<uint32_t>(e8[5]) << 16);
    u.w = e8[6] | (static_cast<uint32_t>(e8[7]) << 16);
    yr[v] = u;
  }
}

inline int launch_pack_hw(const uint16_t* x, uint16_t* y, const uint16_t* w, uint16_t* wy, int64_t rows, int64_t ih,
                          int64_t iw, int64_t c, int64_t oh, int64_t ow, int64_t kh, int64_t kw, int64_t sh,
                          int64_t sw, int64_t ph, int64_t pw, int64_t dh, int64_t dw, int64_t cp, int64_t kd,
                          int64_t co, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(kh * iw * c * 2);
  if (smem > 96 * 1024 || rows >= (1ll << 31) - 64 || cp > 256) return 2;  // caller falls back
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(pack_hw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024) != cudaSuccess)
      return 1;
    attr_set = true;
  }
  const int wblocks = 16;
  pack_hw_kernel<<<static_cast<unsigned>(rows + wblocks), 256, smem, st>>>(
      x, y, w, wy, static_cast<int32_t>(rows), static_cast<int32_t>(ih), static_cast<int32_t>(iw),
      static_cast<int32_t>(c), static_cast<int32_t>(oh), static_cast<int32_t>(ow), static_cast<int32_t>(kh),
      static_cast<int32_t>(kw), static_cast<int32_t>(sh), static_cast<int32_t>(sw), static_cast<int32_t>(ph),
      static_cast<int32_t>(pw), static_cast<int32_t>(dh), static_cast<int32_t>(dw), static_cast<int32_t>(cp),
      static_cast<int32_t>(kd), static_cast<int32_t>(co));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

inline int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return static_cast<int>(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

inline int launch_pad_channels(const uint16_t* x, uint16_t* y, int64_t pixels, int64_t c,
                               int64_t cp, cudaStream_t st) {
  pad_channels_kernel<<<grid_for(pixels * cp), 256, 0, st>>>(x, y, pixels, static_cast<int32_t>(c),
                                                             static_cast<int32_t>(cp));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

inline int launch_pad_weight_rows(const uint16_t* w, uint16_t* y, int64_t taps, int64_t c,
                                  int64_t cp, int64_t co, cudaStream_t st) {
  pad_weight_rows_kernel<<<grid_for(taps * cp * co), 256, 0, st>>>(
      w, y, taps, static_cast<int32_t>(c), static_cast<int32_t>(cp), static_cast<int32_t>(co));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

inline int launch_pack_kw(const uint16_t* x, uint16_t* y, int64_t rows, int64_t iw, int64_t c,
                          int64_t ow, int64_t kw, int64_t sw, int64_t pw, int64_t dw, int64_t cp,
                          cudaStream_t st) {
  pack_kw_kernel<<<grid_for(rows * ow * (cp / 8)), 256, 0, st>>>(
      x, y, rows, static_cast<int32_t>(iw), static_cast<int32_t>(c), static_cast<int32_t>(ow),
      static_cast<int32_t>(kw), static_cast<int32_t>(sw), static_cast<int32_t>(pw),
      static_cast<int32_t>(dw), static_cast<int32_t>(cp));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

inline int launch_pack_kw_weights(const uint16_t* w, uint16_t* y, int64_t khd, int64_t kwc, int64_t cp,
                                  int64_t co, cudaStream_t st) {
  pack_kw_weights_kernel<<<grid_for(khd * cp * co), 256, 0, st>>>(
      w, y, khd, static_cast<int32_t>(kwc), static_cast<int32_t>(cp), static_cast<int32_t>(co));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

inline int launch_f32_to_f16_exact(const float* x, uint16_t* y, int64_t n, int* flag,
                                   cudaStream_t st) {
  f32_to_f16_exact_kernel<<<grid_for(n), 256, 0, st>>>(x, y, n, flag);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace tb
