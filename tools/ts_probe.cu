// ts_probe.cu — probe for an A-from-TMEM (TS) direct convolution on sm_100a:
//   1. tcgen05.cp.128x256b from a SW128 K-major smem window starting at any 128-byte
//      row lands row R0+m in TMEM lane m (checked with tcgen05.ld)
//   2. tcgen05.shift.down moves lane m to lane m+1 (what happens to lane 0)
//   3. a TS MMA (A = the copied window) equals the SS MMA on the same window, bitwise
//   4. the same after a shift: TS on the shifted copy == SS with the descriptor at R0-1
//   5. cycles per 3x3 halo tile (36 MMAs): SS shifted descriptors vs TS cp+shift
// Not part of the product. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ts_probe tools/ts_probe.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2207_04296_b200/csrc/ptx.cuh"

using namespace tb;

__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tcp(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void tshift(uint32_t taddr) {
  asm volatile("tcgen05.shift.cta_group::1.down [%0];" ::"r"(taddr) : "memory");
}

constexpr int kRows = 256;
__device__ __forceinline__ float aval(int r, int k) { return (float)(((r * 7 + k * 3) % 17) - 8) * 0.125f; }
__device__ __forceinline__ float bval(int k, int n) { return (float)(((k * 5 + n * 11) % 13) - 6) * 0.25f; }

// out: [0..] error counters and lane-0 diagnostics
__global__ void probe(int R0, int* out, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                  // kRows x 128 B, SW128
  uint8_t* sB = smem + kRows * 128;    // 64 K rows x 128 B (N = 64), MN-major SW128
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < kRows * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    const int chunk = (k / 8) ^ (r & 7);
    *reinterpret_cast<__half*>(sA + r * 128 + chunk * 16 + (k % 8) * 2) = __float2half(aval(r, k));
  }
  for (int i = tid; i < 64 * 64; i += blockDim.x) {
    const int k = i / 64, n = i % 64;
    const int chunk = (n / 8) ^ (k & 7);
    *reinterpret_cast<__half*>(sB + k * 128 + chunk * 16 + (n % 8) * 2) = __float2half(bval(k, n));
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (tid < 32) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t TA = tmem + 256, TD_SS = tmem + 0, TD_TS = tmem + 64, TD_SS2 = tmem + 128, TD_TS2 = tmem + 192;
  const uint32_t idesc = idesc_f16_f32(128, 64, 0, 1);
  const uint64_t a0 = smem_desc(smem_u32(sA), 16, 1024, 2);
  const uint64_t b0 = smem_desc(smem_u32(sB), 8192, 1024, 2);
  uint32_t phase = 0;
  auto wait_all = [&]() {
    if (tid < 32) {
      if (elect_one()) umma_commit(&bar);
      __syncwarp();
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc_fence_after();
  };
  // 1. cp window at R0 -> TA
  if (tid < 32 && elect_one()) {
    for (int c = 0; c < 4; ++c) tcp(TA + 8 * c, a0 + ((R0 * 128) >> 4) + 2 * c);
    // 3. SS and TS MMAs on the same window
    for (int k = 0; k < 4; ++k) {
      umma_f16(TD_SS, a0 + ((R0 * 128) >> 4) + 2 * k, b0 + 64 * k, idesc, k != 0);
      umma_ts(TD_TS, TA + 8 * k, b0 + 64 * k, idesc, k != 0);
    }
  }
  __syncwarp();
  wait_all();
  const uint32_t q = tid / 32, lane = tid % 32, m = tid;
  int err_cp = 0, err_mma = 0;
  {
    uint32_t r[32];
    tmem_ld_32x32b_x32(TA + ((q * 32u) << 16), r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) {
      const __half2 h = *reinterpret_cast<__half2*>(&r[j]);
      if (__half2float(h.x) != aval(R0 + m, 2 * j) || __half2float(h.y) != aval(R0 + m, 2 * j + 1)) ++err_cp;
    }
    uint32_t d1[32], d2[32];
    for (int c0 = 0; c0 < 64; c0 += 32) {
      tmem_ld_32x32b_x32(TD_SS + ((q * 32u) << 16) + c0, d1);
      tmem_ld_32x32b_x32(TD_TS + ((q * 32u) << 16) + c0, d2);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) err_mma += d1[j] != d2[j];
    }
  }
  // 2./4. shift, then TS on the shifted copy vs SS at R0 - 1
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid < 32 && elect_one()) {
    for (int c = 0; c < 4; ++c) tshift(TA + 8 * c);
    for (int k = 0; k < 4; ++k) {
      umma_f16(TD_SS2, a0 + (((R0 - 1) * 128) >> 4) + 2 * k, b0 + 64 * k, idesc, k != 0);
      umma_ts(TD_TS2, TA + 8 * k, b0 + 64 * k, idesc, k != 0);
    }
  }
  __syncwarp();
  wait_all();
  int err_shift = 0, err_mma2 = 0, lane0_src = -2;
  {
    uint32_t r[32];
    tmem_ld_32x32b_x32(TA + ((q * 32u) << 16), r);
    tmem_ld_wait();
    if (m >= 1) {
      for (int j = 0; j < 32; ++j) {
        const __half2 h = *reinterpret_cast<__half2*>(&r[j]);
        if (__half2float(h.x) != aval(R0 + m - 1, 2 * j) || __half2float(h.y) != aval(R0 + m - 1, 2 * j + 1))
          ++err_shift;
      }
    } else {
      for (int src = 0; src < kRows; ++src) {
        bool ok = true;
        for (int j = 0; j < 32 && ok; ++j) {
          const __half2 h = *reinterpret_cast<__half2*>(&r[j]);
          ok = __half2float(h.x) == aval(src, 2 * j) && __half2float(h.y) == aval(src, 2 * j + 1);
        }
        if (ok) { lane0_src = src; break; }
      }
      if (lane0_src == -2) lane0_src = -1;
    }
    uint32_t d1[32], d2[32];
    for (int c0 = 0; c0 < 64; c0 += 32) {
      tmem_ld_32x32b_x32(TD_SS2 + ((q * 32u) << 16) + c0, d1);
      tmem_ld_32x32b_x32(TD_TS2 + ((q * 32u) << 16) + c0, d2);
      tmem_ld_wait();
      if (m >= 1)
        for (int j = 0; j < 32; ++j) err_mma2 += d1[j] != d2[j];
    }
  }
  atomicAdd(&out[0], err_cp);
  atomicAdd(&out[1], err_mma);
  atomicAdd(&out[2], err_shift);
  atomicAdd(&out[3], err_mma2);
  if (m == 0) out[4] = lane0_src;
  // 5. timing: 3x3 halo tile sequences, Wv = 58
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int tiles = 64;
  for (int mode = 0; mode < 2; ++mode) {
    unsigned long long t0 = clock64();
    if (tid < 32 && elect_one()) {
      for (int t = 0; t < tiles; ++t) {
        const uint32_t D = tmem + 64 * (t & 1);
        for (int ty = 0; ty < 3; ++ty) {
          if (mode == 0) {
#pragma unroll
            for (int tx = 0; tx < 3; ++tx)
#pragma unroll
              for (int k = 0; k < 4; ++k)
                umma_f16(D, a0 + (((ty * 58 + tx) * 128) >> 4) + 2 * k, b0 + 64 * k, idesc, 1);
          } else {
            const uint32_t A = TA + 32 * ty;
#pragma unroll
            for (int c = 0; c < 4; ++c) tcp(A + 8 * c, a0 + (((ty * 58) * 128) >> 4) + 2 * c);
#pragma unroll
            for (int tx = 0; tx < 3; ++tx) {
              if (tx) {
#pragma unroll
                for (int c = 0; c < 4; ++c) tshift(A + 8 * c);
              }
#pragma unroll
              for (int k = 0; k < 4; ++k) umma_ts(D, A + 8 * k, b0 + 64 * k, idesc, 1);
            }
          }
        }
      }
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, phase);
    phase ^= 1;
    unsigned long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x * 2 + mode] = (t1 - t0) / tiles;
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tmem, 512);
}

int main() {
  int* d;
  unsigned long long* c;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 148 * 2 * 8);
  const int smem = kRows * 128 + 64 * 128 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int R0 : {1, 5, 58, 61}) {
    cudaMemset(d, 0, 64);
    probe<<<148, 128, smem>>>(R0, d, c);
    cudaError_t e = cudaDeviceSynchronize();
    int h[5];
    unsigned long long hc[2];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, c, sizeof hc, cudaMemcpyDeviceToHost);
    printf("R0=%3d cp_err %d  ts_vs_ss_err %d  shift_err(lanes>=1) %d  ts_vs_ss_after_shift_err %d  lane0 after shift = row %d  "
           "| cycles/tile SS %llu  TS(cp+shift) %llu  %s\n",
           R0, h[0] / 148, h[1] / 148, h[2] / 148, h[3] / 148, h[4], hc[0], hc[1], e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
