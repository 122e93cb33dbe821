// dep.cuh — depthwise convolution (DEP) on CUDA cores, HBM-bound.
//
// Semantics: depthwise_source (/root/reference/proj/tests/testing/workloads.h:133-166)
// generalised to batch / stride / padding / dilation: Y[n,oh,ow,c] (+)=
// sum_{rh,rw} X[n, oh*s-p+rh*d, ow*s-p+rw*d, c] * W[rh,rw,c].
// Accumulation is fp32 from 0.0 (or Yin) in the reference's (rh, rw) loop order
// with explicitly separate round-to-nearest multiply and add (__fmul_rn /
// __fadd_rn: the interpreter evaluates mul and add as two rounded fp32 ops,
// src/interp.cc:484-512). Padded taps are skipped (the oracle adds 0*w, which
// leaves a non-negative-zero accumulator unchanged), so the result equals the
// oracle's for ANY fp16 input, not only on the reference distribution.
//
// Layout: each thread owns VEC consecutive channels (one 16-byte fp16 vector for
// VEC = 8) of R vertically adjacent output pixels, so the (R-1)*s + KH input
// rows it touches are loaded once per column tap and reused across the R
// outputs. A warp spans consecutive channel vectors then consecutive output
// columns, so every load and store is a fully coalesced 16/32-byte vector.
#pragma once

#include "ptx.cuh"

namespace tb {

struct DepParams {
  const __half* X;
  const __half* W;
  const float* Yin;
  void* Y;
  int32_t n, ih, iw, c, oh, ow;
  int32_t kh, kw, sh, sw, ph, pw, dh, dw;
  int32_t accumulate, out_f16;
};

template <int VEC, int R>
__global__ void __launch_bounds__(256) dep_kernel(const DepParams p) {
  // 32-bit index math (the host guarantees n*ceil(oh/R)*ow*c/VEC < 2^31).
  const int cvecs = p.c / VEC;
  const int ohb = (p.oh + R - 1) / R;
  const int total = p.n * ohb * p.ow * cvecs;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int cv = idx % cvecs;
    int rest = idx / cvecs;
    const int ox = rest % p.ow;
    rest /= p.ow;
    const int oyb = rest % ohb;
    const int n = rest / ohb;
    const int oy0 = oyb * R;
    const int c0 = cv * VEC;

    float acc[R][VEC];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[r][v] = 0.0f;
    if (p.accumulate) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (oy0 + r >= p.oh) break;
        const float* yin = p.Yin + ((static_cast<int64_t>(n) * p.oh + oy0 + r) * p.ow + ox) * p.c + c0;
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[r][v] = yin[v];
      }
    }

    const __half* xn = p.X + static_cast<int64_t>(n) * p.ih * p.iw * p.c + c0;
    for (int rh = 0; rh < p.kh; ++rh) {
      for (int rw = 0; rw < p.kw; ++rw) {
        float w[VEC];
        const __half* wp = p.W + (rh * p.kw + rw) * p.c + c0;
        if constexpr (VEC == 8) {
          uint4 u = __ldg(reinterpret_cast<const uint4*>(wp));
          const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            float2 f = __half22float2(h[v]);
            w[2 * v] = f.x;
            w[2 * v + 1] = f.y;
          }
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) w[v] = __half2float(wp[v]);
        }
        const int ix = ox * p.sw - p.pw + rw * p.dw;
        if (ix < 0 || ix >= p.iw) continue;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int oy = oy0 + r;
          if (oy >= p.oh) break;
          const int iy = oy * p.sh - p.ph + rh * p.dh;
          if (iy < 0 || iy >= p.ih) continue;
          const __half* xp = xn + (static_cast<int64_t>(iy) * p.iw + ix) * p.c;
          float x[VEC];
          if constexpr (VEC == 8) {
            uint4 u = __ldg(reinterpret_cast<const uint4*>(xp));
            const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float2 f = __half22float2(h[v]);
              x[2 * v] = f.x;
              x[2 * v + 1] = f.y;
            }
          } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) x[v] = __half2float(xp[v]);
          }
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc[r][v] = __fadd_rn(acc[r][v], __fmul_rn(x[v], w[v]));
        }
      }
    }

#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int oy = oy0 + r;
      if (oy >= p.oh) break;
      const int64_t off = ((static_cast<int64_t>(n) * p.oh + oy) * p.ow + ox) * p.c + c0;
      if (p.out_f16) {
        __half* y = reinterpret_cast<__half*>(p.Y) + off;
        if constexpr (VEC == 8) {
          uint4 u;
          __half2 h[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) h[v] = __floats2half2_rn(acc[r][2 * v], acc[r][2 * v + 1]);
          u.x = *reinterpret_cast<uint32_t*>(&h[0]);
          u.y = *reinterpret_cast<uint32_t*>(&h[1]);
          u.z = *reinterpret_cast<uint32_t*>(&h[2]);
          u.w = *reinterpret_cast<uint32_t*>(&h[3]);
          *reinterpret_cast<uint4*>(y) = u;
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) y[v] = __float2half_rn(acc[r][v]);
        }
      } else {
        float* y = reinterpret_cast<float*>(p.Y) + off;
        if constexpr (VEC == 8) {
          reinterpret_cast<float4*>(y)[0] = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
          reinterpret_cast<float4*>(y)[1] = make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]);
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) y[v] = acc[r][v];
        }
      }
    }
  }
}

}  // namespace tb
