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

// ---------------------------------------------------------------------------
// dep_tile_kernel — the fast path for K x K depthwise with compile-time stride.
//
// Block = TR x TC output pixels x 32 channels (128 threads). Its input footprint
// ((TR-1)S + K rows x (TC-1)S + K cols x 32 ch, fp16) arrives in smem as ONE
// 4-D TMA box; out-of-bounds coordinates are zero-filled, which is exactly the
// reference's select(in-bounds, x, 0.0) padding (the oracle then adds 0*w, and
// so does this kernel — bit-identical, including signed zeros).
// Thread = R x T output pixels x 8 channels with all K*K*8 weights in
// registers. It walks its input footprint ONCE in row-major order and adds
// x * w[iy - r*S][ix - t*S] to every output that uses that pixel: for a fixed
// output, row-major (iy, ix) visits taps in row-major (rh, rw) order — the
// reference's reduction order — so results are bit-exact for any input.
// Smem reads per output: (R-1)S+K)((T-1)S+K)/(R*T) instead of K*K.
struct DepTileParams {
  CUtensorMap tmX;  // 4-D over X[N, H, W, C]: box {32, FC, FR, 1}
  const __half* W;
  const float* Yin;
  void* Y;
  int32_t n, c, oh, ow, pad_h, pad_w;
  int32_t tiles_h, tiles_w, cblocks;
  int32_t accumulate, out_f16;
};

template <int K, int S, int R, int T, int TR, int TC>
__global__ void __launch_bounds__(128) dep_tile_kernel(const __grid_constant__ DepTileParams p) {
  constexpr int FR = (TR - 1) * S + K, FC = (TC - 1) * S + K;  // block footprint
  constexpr int fr = (R - 1) * S + K, fc = (T - 1) * S + K;    // thread footprint
  constexpr int CT = 32;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __half* tile = reinterpret_cast<__half*>(smem_raw);
  __shared__ __align__(8) uint64_t bar;

  int b = blockIdx.x;
  const int cb = b % p.cblocks;
  b /= p.cblocks;
  const int tw = b % p.tiles_w;
  b /= p.tiles_w;
  const int th = b % p.tiles_h;
  const int n = b / p.tiles_h;
  const int oy0 = th * TR, ox0 = tw * TC, c0 = cb * CT;

  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, FR * FC * CT * 2);
    tma_load_4d(tile, &p.tmX, &bar, c0, ox0 * S - p.pad_w, oy0 * S - p.pad_h, n);
  }
  const int cv = threadIdx.x % 4;               // 8-channel vector
  const int tc = (threadIdx.x / 4) % (TC / T);  // thread column
  const int tr = threadIdx.x / (4 * (TC / T));  // thread row
  // weights -> registers while the tile is in flight
  float w[K][K][8];
#pragma unroll
  for (int rh = 0; rh < K; ++rh)
#pragma unroll
    for (int rw = 0; rw < K; ++rw) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(p.W + (rh * K + rw) * p.c + c0 + cv * 8));
      const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const float2 f = __half22float2(h[v]);
        w[rh][rw][2 * v] = f.x;
        w[rh][rw][2 * v + 1] = f.y;
      }
    }
  float acc[R][T][8];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int oy = oy0 + tr * R + r, ox = ox0 + tc * T + t;
      const bool in = oy < p.oh && ox < p.ow;
      if (p.accumulate && in) {
        const float* yin = p.Yin + ((static_cast<int64_t>(n) * p.oh + oy) * p.ow + ox) * p.c + c0 + cv * 8;
        const float4 a = *reinterpret_cast<const float4*>(yin);
        const float4 bb = *reinterpret_cast<const float4*>(yin + 4);
        acc[r][t][0] = a.x; acc[r][t][1] = a.y; acc[r][t][2] = a.z; acc[r][t][3] = a.w;
        acc[r][t][4] = bb.x; acc[r][t][5] = bb.y; acc[r][t][6] = bb.z; acc[r][t][7] = bb.w;
      } else {
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[r][t][v] = 0.0f;
      }
    }
  mbar_wait(&bar, 0);
  const __half* my = tile + ((tr * R * S) * FC + tc * T * S) * CT + cv * 8;
#pragma unroll
  for (int iy = 0; iy < fr; ++iy) {
#pragma unroll
    for (int ix = 0; ix < fc; ++ix) {
      const uint4 u = *reinterpret_cast<const uint4*>(my + (iy * FC + ix) * CT);
      const __half2* h = reinterpret_cast<const __half2*>(&u);
      float x[8];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const float2 f = __half22float2(h[v]);
        x[2 * v] = f.x;
        x[2 * v + 1] = f.y;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int rh = iy - r * S;
        if (rh < 0 || rh >= K) continue;
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int rw = ix - t * S;
          if (rw < 0 || rw >= K) continue;
#pragma unroll
          for (int v = 0; v < 8; ++v)
            acc[r][t][v] = __fadd_rn(acc[r][t][v], __fmul_rn(x[v], w[rh][rw][v]));
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int oy = oy0 + tr * R + r, ox = ox0 + tc * T + t;
      if (oy >= p.oh || ox >= p.ow) continue;
      const int64_t off = ((static_cast<int64_t>(n) * p.oh + oy) * p.ow + ox) * p.c + c0 + cv * 8;
      if (p.out_f16) {
        uint4 u;
        __half2 hh[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) hh[v] = __floats2half2_rn(acc[r][t][2 * v], acc[r][t][2 * v + 1]);
        u.x = *reinterpret_cast<uint32_t*>(&hh[0]);
        u.y = *reinterpret_cast<uint32_t*>(&hh[1]);
        u.z = *reinterpret_cast<uint32_t*>(&hh[2]);
        u.w = *reinterpret_cast<uint32_t*>(&hh[3]);
        *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(p.Y) + off) = u;
      } else {
        float* y = reinterpret_cast<float*>(p.Y) + off;
        reinterpret_cast<float4*>(y)[0] = make_float4(acc[r][t][0], acc[r][t][1], acc[r][t][2], acc[r][t][3]);
        reinterpret_cast<float4*>(y)[1] = make_float4(acc[r][t][4], acc[r][t][5], acc[r][t][6], acc[r][t][7]);
      }
    }
}

}  // namespace tb
