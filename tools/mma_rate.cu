// mma_rate.cu — microbenchmark: tcgen05.mma (kind::f16, cta_group::1, SS)
// throughput per SM by N and A-operand row alignment, operands resident in
// smem (no TMA). Reports cycles per MMA (M=128, K=16). Not part of the product.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2207_04296_b200/csrc/ptx.cuh"

using namespace tb;

template <int N>
__global__ void mma_kernel(int iters, int a_row_step, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  // zero operands (values irrelevant)
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) { tmem_alloc(&tslot, 256); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint64_t a0 = smem_desc(smem_u32(smem), 16, 1024, 2);
    const uint64_t b0 = smem_desc(smem_u32(smem + 64 * 1024), 8192, 1024, 2);
    const uint32_t idesc = idesc_f16_f32(128, N, 0, 1);
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < iters; ++i) {
        const uint32_t row = (i * a_row_step) & 127;
        umma_f16(tmem, a0 + ((row * 128) >> 4) + 2 * (i & 3), b0 + 128 * (i & 3), idesc, 1);
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
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

template <int N>
void run(int grid, int a_row_step) {
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  cudaFuncSetAttribute(mma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  mma_kernel<N><<<grid, 128, 100 * 1024>>>(iters, a_row_step, d);
  mma_kernel<N><<<grid, 128, 100 * 1024>>>(iters, a_row_step, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  printf("N=%3d grid=%3d A row step %2d: %.1f cycles/MMA (ideal %d) %s\n", N, grid, a_row_step,
         avg / iters, N / 2, e ? cudaGetErrorString(e) : "");
  cudaFree(d);
}

int main() {
  for (int step : {0, 1, 8}) {
    run<64>(1, step);
    run<64>(148, step);
  }
  run<32>(148, 0);
  run<128>(148, 0);
  run<128>(148, 1);
  run<256>(148, 0);
  return 0;
}
