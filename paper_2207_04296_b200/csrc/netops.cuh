// netops.cuh — the non-contraction glue of the network graphs (SURVEY §8(f)
// row 3): NHWC fp16 max pooling, global average pooling, row LayerNorm and row
// softmax. All are single-pass HBM-bound CUDA-core kernels with 16-byte vector
// accesses along the contiguous channel / feature dim; the contractions of the
// networks (every conv and GEMM, with bias / residual / activation fused into
// their epilogues) run on the tcgen05 kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tb {

union H8 {
  uint4 u;
  __half2 h[4];
};

// Y[n, oy, ox, c] = max over the k x k window (stride s, pad p; padding never
// wins, as in torch's max_pool2d). Thread = one 8-channel vector of one output pixel.
__global__ void maxpool2d_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y, int n, int h,
                                 int w, int c, int oh, int ow, int k, int s, int p) {
  const int cv = c / 8;
  const int64_t total = static_cast<int64_t>(n) * oh * ow * cv;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int v = static_cast<int>(i % cv);
    int64_t r = i / cv;
    const int ox = static_cast<int>(r % ow);
    r /= ow;
    const int oy = static_cast<int>(r % oh);
    const int b = static_cast<int>(r / oh);
    H8 m;
    const __half2 ninf = __half2half2(__ushort_as_half(0xFC00));
    for (int j = 0; j < 4; ++j) m.h[j] = ninf;
    for (int ky = 0; ky < k; ++ky) {
      const int iy = oy * s - p + ky;
      if (iy < 0 || iy >= h) continue;
      for (int kx = 0; kx < k; ++kx) {
        const int ix = ox * s - p + kx;
        if (ix < 0 || ix >= w) continue;
        H8 x;
        x.u = __ldg(reinterpret_cast<const uint4*>(X + ((static_cast<int64_t>(b) * h + iy) * w + ix) * c) + v);
        for (int j = 0; j < 4; ++j) m.h[j] = __hmax2(m.h[j], x.h[j]);
      }
    }
    reinterpret_cast<uint4*>(Y + ((static_cast<int64_t>(b) * oh + oy) * ow + ox) * c)[v] = m.u;
  }
}

// Y[n, c] = fp16(sum_{hw} X[n, hw, c] / hw), fp32 sum in pixel order.
// Block = (image, 256 channel vectors of 8); threads stride the pixels.
__global__ void avgpool_global_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y, int hw,
                                      int c) {
  const int cv = c / 8;
  const int b = blockIdx.y;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= cv) return;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const uint4* src = reinterpret_cast<const uint4*>(X + static_cast<int64_t>(b) * hw * c) + v;
  for (int i = 0; i < hw; ++i) {
    H8 x;
    x.u = __ldg(src + static_cast<int64_t>(i) * cv);
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(x.h[j]);
      acc[2 * j] += f.x;
      acc[2 * j + 1] += f.y;
    }
  }
  H8 o;
  const float inv = 1.0f / static_cast<float>(hw);
  for (int j = 0; j < 4; ++j) o.h[j] = __floats2half2_rn(acc[2 * j] * inv, acc[2 * j + 1] * inv);
  reinterpret_cast<uint4*>(Y + static_cast<int64_t>(b) * c)[v] = o.u;
}

__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.f;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

__device__ __forceinline__ float block_max(float v, float* red) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = -INFINITY;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) t = fmaxf(t, red[i]);
  return t;
}

// Y[r, :] = (X[r, :] - mean) * rsqrt(var + eps) * gamma + beta; one block per row,
// the row held in registers (cols / 8 / blockDim vectors per thread, <= 4).
template <int VPT>
__global__ void layernorm_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y,
                                 const float* __restrict__ gamma, const float* __restrict__ beta, int cols,
                                 float eps) {
  __shared__ float red[32];
  const int cv = cols / 8;
  const uint4* x = reinterpret_cast<const uint4*>(X + static_cast<int64_t>(blockIdx.x) * cols);
  float v[VPT][8];
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < VPT; ++t) {
    const int i = threadIdx.x + t * blockDim.x;
    if (i < cv) {
      H8 h;
      h.u = __ldg(x + i);
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(h.h[j]);
        v[t][2 * j] = f.x;
        v[t][2 * j + 1] = f.y;
        sum += f.x + f.y;
      }
    } else {
      for (int j = 0; j < 8; ++j) v[t][j] = 0.f;
    }
  }
  const float mean = block_sum(sum, red) / cols;
  float sq = 0.f;
#pragma unroll
  for (int t = 0; t < VPT; ++t) {
    const int i = threadIdx.x + t * blockDim.x;
    if (i < cv)
      for (int j = 0; j < 8; ++j) sq += (v[t][j] - mean) * (v[t][j] - mean);
  }
  const float rstd = rsqrtf(block_sum(sq, red) / cols + eps);
  uint4* y = reinterpret_cast<uint4*>(Y + static_cast<int64_t>(blockIdx.x) * cols);
#pragma unroll
  for (int t = 0; t < VPT; ++t) {
    const int i = threadIdx.x + t * blockDim.x;
    if (i >= cv) continue;
    H8 o;
    for (int j = 0; j < 4; ++j) {
      const int c0 = i * 8 + 2 * j;
      const float a = (v[t][2 * j] - mean) * rstd * __ldg(gamma + c0) + __ldg(beta + c0);
      const float b = (v[t][2 * j + 1] - mean) * rstd * __ldg(gamma + c0 + 1) + __ldg(beta + c0 + 1);
      o.h[j] = __floats2half2_rn(a, b);
    }
    y[i] = o.u;
  }
}

// Y[r, :] = softmax(scale * X[r, :]) in fp32, written fp16; one block per row.
template <int VPT>
__global__ void softmax_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y, int cols, float scale) {
  __shared__ float red[32];
  const int cv = cols / 8;
  const uint4* x = reinterpret_cast<const uint4*>(X + static_cast<int64_t>(blockIdx.x) * cols);
  float v[VPT][8];
  float mx = -INFINITY;
#pragma unroll
  for (int t = 0; t < VPT; ++t) {
    const int i = threadIdx.x + t * blockDim.x;
    if (i < cv) {
      H8 h;
      h.u = __ldg(x + i);
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(h.h[j]);
        v[t][2 * j] = f.x * scale;
        v[t][2 * j + 1] = f.y * scale;
        mx = fmaxf(mx, fmaxf(v[t][2 * j], v[t][2 * j + 1]));
      }
    }
  }
  mx = block_max(mx, red);
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < VPT; ++t) {
    const int i = threadIdx.x + t * blockDim.x;
    if (i < cv)
      for (int j = 0; j < 8; ++j) {
        v[t][j] = __expf(v[t][j] - mx);
        sum += v[t][j];
      }
  }
  const float inv = 1.0f / block_sum(sum, red);
  uint4* y = reinterpret_cast<uint4*>(Y + static_cast<int64_t>(blockIdx.x) * cols);
#pragma unroll
  for (int t = 0; t < VPT; ++t) {
    const int i = threadIdx.x + t * blockDim.x;
    if (i >= cv) continue;
    H8 o;
    for (int j = 0; j < 4; ++j) o.h[j] = __floats2half2_rn(v[t][2 * j] * inv, v[t][2 * j + 1] * inv);
    y[i] = o.u;
  }
}

// Warp-per-row variants (cols <= 256 * VPL, the BERT shapes: 512-wide softmax
// rows, 1024-wide LayerNorm rows): the row lives in one warp's registers,
// reductions are shuffles, no block barriers, 8 rows per 256-thread block.
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int VPL>
__global__ void __launch_bounds__(256) softmax_warp_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y,
                                                           int rows, int cols, float scale) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int cv = cols / 8;
  const uint4* x = reinterpret_cast<const uint4*>(X + static_cast<int64_t>(row) * cols);
  float v[VPL][8];
  float mx = -INFINITY;
#pragma unroll
  for (int t = 0; t < VPL; ++t) {
    const int i = lane + 32 * t;
    if (i < cv) {
      H8 h;
      h.u = __ldg(x + i);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(h.h[j]);
        v[t][2 * j] = f.x * scale;
        v[t][2 * j + 1] = f.y * scale;
        mx = fmaxf(mx, fmaxf(v[t][2 * j], v[t][2 * j + 1]));
      }
    }
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < VPL; ++t) {
    if (lane + 32 * t < cv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[t][j] = __expf(v[t][j] - mx);
        sum += v[t][j];
      }
    }
  }
  const float inv = 1.0f / warp_sum(sum);
  uint4* y = reinterpret_cast<uint4*>(Y + static_cast<int64_t>(row) * cols);
#pragma unroll
  for (int t = 0; t < VPL; ++t) {
    const int i = lane + 32 * t;
    if (i >= cv) continue;
    H8 o;
#pragma unroll
    for (int j = 0; j < 4; ++j) o.h[j] = __floats2half2_rn(v[t][2 * j] * inv, v[t][2 * j + 1] * inv);
    y[i] = o.u;
  }
}

template <int VPL>
__global__ void __launch_bounds__(256) layernorm_warp_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y,
                                                             const float* __restrict__ gamma,
                                                             const float* __restrict__ beta, int rows, int cols,
                                                             float eps) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int cv = cols / 8;
  const uint4* x = reinterpret_cast<const uint4*>(X + static_cast<int64_t>(row) * cols);
  float v[VPL][8];
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < VPL; ++t) {
    const int i = lane + 32 * t;
    if (i < cv) {
      H8 h;
      h.u = __ldg(x + i);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(h.h[j]);
        v[t][2 * j] = f.x;
        v[t][2 * j + 1] = f.y;
        sum += f.x + f.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[t][j] = 0.f;
    }
  }
  const float mean = warp_sum(sum) / cols;
  float sq = 0.f;
#pragma unroll
  for (int t = 0; t < VPL; ++t)
    if (lane + 32 * t < cv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) sq += (v[t][j] - mean) * (v[t][j] - mean);
    }
  const float rstd = rsqrtf(warp_sum(sq) / cols + eps);
  uint4* y = reinterpret_cast<uint4*>(Y + static_cast<int64_t>(row) * cols);
#pragma unroll
  for (int t = 0; t < VPL; ++t) {
    const int i = lane + 32 * t;
    if (i >= cv) continue;
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma) + 2 * i);
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma) + 2 * i + 1);
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta) + 2 * i);
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta) + 2 * i + 1);
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    H8 o;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      o.h[j] = __floats2half2_rn((v[t][2 * j] - mean) * rstd * g[2 * j] + b[2 * j],
                                 (v[t][2 * j + 1] - mean) * rstd * g[2 * j + 1] + b[2 * j + 1]);
    y[i] = o.u;
  }
}

}  // namespace tb

