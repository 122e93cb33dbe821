// mma_rate2.cu — microbenchmark: tcgen05.mma kind::f16 M=128 K=16 issue rate per SM
// for the operand sources a direct convolution could use:
//   SS  : A and B from shared memory (B MN-major or K-major)
//   TS  : A from tensor memory, B from shared memory
// plus tcgen05.st / tcgen05.cp throughput (filling A in TMEM).
// Not part of the product. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate2 tools/mma_rate2.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2207_04296_b200/csrc/ptx.cuh"

using namespace tb;

__device__ __forceinline__ void umma_ts_(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                         uint32_t acc);
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_ts_(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                         uint32_t acc) {
  umma_ts(tmem_d, tmem_a, bdesc, idesc, acc);
}

// mode 0: SS B MN-major, 1: SS B K-major, 2: TS B MN-major, 3: TS B K-major
template <int N, int MODE>
__global__ void mma_kernel(int iters, int a_row_step, unsigned long long* out) {
  constexpr int mode = MODE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint64_t a0 = smem_desc(smem_u32(smem), 16, 1024, 2);
    constexpr bool kmaj = mode & 1;
    // B MN-major: 128-byte rows along N, K rows (SBO 8 rows); K-major: N rows of 128 B (K 64)
    const uint64_t b0 = kmaj ? smem_desc(smem_u32(smem + 64 * 1024), 16, 1024, 2)
                             : smem_desc(smem_u32(smem + 64 * 1024), 8192, 1024, 2);
    const uint32_t idesc = idesc_f16_f32(128, N, 0, kmaj ? 0 : 1);
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < iters; ++i) {
        const uint32_t row = (i * a_row_step) & 127;
        const uint64_t bd = kmaj ? b0 + 2 * (i & 3) : b0 + 128 * (i & 3);
        if constexpr (mode < 2)
          umma_f16(tmem, a0 + ((row * 128) >> 4) + 2 * (i & 3), bd, idesc, 1);
        else
          umma_ts(tmem, tmem + 256 + 8 * (i & 7), bd, idesc, 1);
      }
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// tcgen05.st 32x32b.x32 from 4 warps (each its lane quadrant): bytes per cycle into TMEM
__global__ void tmem_st_kernel(int iters, unsigned long long* out) {
  __shared__ uint32_t tslot;
  if (threadIdx.x < 32) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t q = threadIdx.x / 32;
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 7 + i;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t addr = tmem + ((q * 32u) << 16) + 32 * (it & 15);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}


__device__ __forceinline__ void tmem_st_n32_(uint32_t t, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(t),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}

// rowpack-like TS MMA stream: per "plane" 4 accumulators x 10 K16 steps, B walks a
// 140 KB panel (7 kd chunks); warps 4..11 optionally load shared memory (lds=1) or
// store 80 TMEM columns (st=1) per plane like the builders.
__global__ void rp_like(int planes, int lds, int st, int ld, unsigned long long* out, int fence = 0, int rnd = 0) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  __shared__ __align__(8) uint64_t bar2;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) {
    uint32_t h = rnd ? (i * 2654435761u) ^ (i >> 3) : 0u;
    // random fp16 pairs in [-2, 2) (exponent bits bounded), or zeros
    uint32_t v = rnd ? ((h & 0x83FF83FFu) | 0x3C003C00u) : 0u;
    ((uint4*)smem)[i] = make_uint4(v, v ^ 0x00050003u, v ^ 0x01100220u, v ^ 0x80008000u);
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_barrier_init(); stop = 0; }
  if (threadIdx.x < 32) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int warp = threadIdx.x / 32;
  if (rnd && warp < 4) {  // random A buffers in TMEM
    uint32_t w[32];
    for (int i = 0; i < 32; ++i) {
      uint32_t h = (threadIdx.x * 97u + i * 2654435761u);
      w[i] = (h & 0x83FF83FFu) | 0x3C003C00u;
    }
    for (int c = 0; c < 160; c += 32) tmem_st_n32_(tmem + ((warp * 32u) << 16) + 320 + c, w);
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const uint64_t b0 = smem_desc(smem_u32(smem), 143360, 1024, 2);
    const uint32_t idesc = idesc_f16_f32(128, 64, 0, 1);
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int pl = 0; pl < planes; ++pl) {
        const uint32_t a = tmem + 320 + 80 * (pl & 1);
        if (fence & 1) tc_fence_after();
        if (fence & 4) umma_commit(&bar2);
        for (int j = 0; j < 4; ++j) {
          if (fence & 2) tc_fence_after();
          const uint32_t d = tmem + 64 * ((pl + j) % 5);
          const uint64_t bk = b0 + ((pl + j) % 7) * ((160 * 128) >> 4);
#pragma unroll
          for (int s = 0; s < 10; ++s) umma_ts_(d, a + 8 * s, bk + s * 128, idesc, 1);
        }
      }
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = (t1 - t0) / planes; stop = 1; }
  } else if (warp >= 4 && warp < 12) {
    const uint32_t base = smem_u32(smem) + 143360 + (threadIdx.x & 31) * 12;
    uint32_t acc = 0;
    const uint32_t q = warp & 3;
    while (!stop) {
      if (lds) {
#pragma unroll 4
        for (int i = 0; i < 48; ++i) {
          uint32_t v;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + 4 * (i % 12) + 240 * (i / 12)));
          acc += v;
        }
      }
      if (st) {
        uint32_t w[8];
        for (int i = 0; i < 8; ++i) w[i] = acc + i;
        for (int c = 0; c < 40; c += 8) {
          const uint32_t ta = tmem + ((q * 32u) << 16) + 320 + 80 * (acc & 1) + (warp >= 8 ? 40 : 0) + c;
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
                       "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
      }
      if (lds < 2) __nanosleep(100);
    }
    if (acc == 12345) out[1000] = acc;
  } else if (warp < 4 && ld) {
    // epilogue-like: read 64 accumulator columns of the lane quadrant, ~one od per 500 cycles
    uint32_t acc = 0;
    while (!stop) {
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + ((warp * 32u) << 16) + 64 * (acc % 5) + c0, r);
        tmem_ld_wait();
        for (int i = 0; i < 32; ++i) acc += r[i];
      }
      __nanosleep(200);
    }
    if (acc == 12345) out[1001] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N, int mode>
void run(int grid, int step) {
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  cudaFuncSetAttribute(mma_kernel<N, mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  mma_kernel<N, mode><<<grid, 128, 100 * 1024>>>(iters, step, d);
  mma_kernel<N, mode><<<grid, 128, 100 * 1024>>>(iters, step, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  static const char* names[] = {"SS B MN-major", "SS B K-major", "TS B MN-major", "TS B K-major"};
  printf("N=%3d grid=%3d %-14s A step %d: %.1f cycles/MMA %s\n", N, grid, names[mode], step, avg / iters,
         e ? cudaGetErrorString(e) : "");
  cudaFree(d);
}

int main() {
  run<64, 0>(148, 1); run<128, 0>(148, 1); run<256, 0>(148, 0);
  run<64, 1>(148, 1); run<128, 1>(148, 1); run<256, 1>(148, 0);
  run<64, 2>(148, 1); run<128, 2>(148, 1); run<256, 2>(148, 0);
  run<64, 3>(148, 1); run<128, 3>(148, 1); run<256, 3>(148, 0);
  run<32, 2>(148, 0);
  {
    unsigned long long* d;
    cudaMalloc(&d, 2000 * 8);
    cudaFuncSetAttribute(rp_like, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rnd = 0; rnd < 2; ++rnd) {
      for (int pl : {256, 20000}) {
        rp_like<<<148, 384, 200 * 1024>>>(pl, 0, 0, 0, d, 0, rnd);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        printf("rowpack-like plane, %s operands, %d planes: %.0f cycles/plane %s\n", rnd ? "random" : "zero", pl,
               avg / 148, e ? cudaGetErrorString(e) : "");
      }
    }
    for (int fence = 1; fence < 2; ++fence) {
      rp_like<<<148, 384, 200 * 1024>>>(256, 0, 0, 0, d, fence);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      printf("rowpack-like plane, fence::after per plane %d per depth %d, commit per plane %d: %.0f cycles/plane %s\n",
             fence & 1, (fence >> 1) & 1, fence >> 2, avg / 148, e ? cudaGetErrorString(e) : "");
    }
    for (int cfg = 0; cfg < 8; ++cfg) {
      const int lds = cfg == 6 ? 2 : cfg == 7 ? 2 : cfg & 1, st = cfg == 7 ? 1 : (cfg >> 1) & 1, ld = cfg == 7 ? 1 : (cfg >> 2) & 1;
      rp_like<<<148, 384, 200 * 1024>>>(cfg == 7 ? 60000 : 256, lds, st, ld, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      printf("rowpack-like plane (40 TS MMAs, 4 accumulators, B over 7 chunks) lds=%d st=%d ld=%d: %.0f cycles/plane (ideal 1280) %s\n",
             lds, st, ld, avg / 148, e ? cudaGetErrorString(e) : "");
    }
  }
  {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int iters = 4096;
    tmem_st_kernel<<<148, 128>>>(iters, d);
    tmem_st_kernel<<<148, 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("tcgen05.st 32x32b.x32 x 4 warps: %.1f cycles per 16 KB (%.1f B/clk) %s\n", avg / iters,
           16384.0 * iters / avg, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
