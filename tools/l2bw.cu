// l2bw.cu — microbenchmark: L2->SM read bandwidth (LDG.128 and cp.async.bulk)
// and HBM read bandwidth, to set the roofline for kernels that re-read operands
// from L2 (im2col taps, halo tiles). Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw tools/l2bw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void ldg_kernel(const int4* __restrict__ p, size_t n_vec, int iters, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_vec;
         i += (size_t)gridDim.x * blockDim.x) {
      int4 v = __ldcg(p + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Each CTA streams `chunk`-byte bulk copies into a ring of `stages` smem slots.
__global__ void bulk_kernel(const char* __restrict__ src, size_t bytes, int chunk, int stages,
                            int iters) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t bars[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = bytes / chunk;
  uint32_t phase[16] = {0};
  int issued = 0, done = 0;
  const size_t total = (size_t)iters * ((nchunks + gridDim.x - 1 - blockIdx.x) / gridDim.x);
  size_t next = blockIdx.x;
  auto issue = [&](int slot) {
    const char* s = src + (next % nchunks) * chunk;
    next += gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[slot])),
                 "r"(chunk)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + (size_t)slot * chunk)),
        "l"(s), "r"(chunk), "r"(smem_u32(&bars[slot]))
        : "memory");
  };
  for (; issued < stages && (size_t)issued < total; ++issued) issue(issued);
  while ((size_t)done < total) {
    const int slot = done % stages;
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P;}"
          : "=r"(ok)
          : "r"(smem_u32(&bars[slot])), "r"(phase[slot])
          : "memory");
    }
    phase[slot] ^= 1;
    ++done;
    if ((size_t)issued < total) {
      issue(slot);
      ++issued;
    }
  }
}

// W producer warps per CTA, each lane 0 running its own ring of `stages` slots.
__global__ void bulk_multi_kernel(const char* __restrict__ src, size_t bytes, int chunk, int stages,
                                  int iters) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t bars[8][8];
  const int w = threadIdx.x / 32, nw = blockDim.x / 32;
  if (threadIdx.x % 32 == 0) {
    for (int i = 0; i < stages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[w][i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x % 32 != 0) return;
  char* my = smem + (size_t)w * stages * chunk;
  const size_t nchunks = bytes / chunk;
  const size_t gid = blockIdx.x * nw + w, gstride = (size_t)gridDim.x * nw;
  uint32_t phase[8] = {0};
  size_t total = (size_t)iters * ((nchunks + gstride - 1 - gid) / gstride), issued = 0, done = 0;
  size_t next = gid;
  auto issue = [&](int slot) {
    const char* s = src + (next % nchunks) * chunk;
    next += gstride;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[w][slot])),
                 "r"(chunk) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(my + (size_t)slot * chunk)), "l"(s), "r"(chunk), "r"(smem_u32(&bars[w][slot])) : "memory");
  };
  for (; issued < (size_t)stages && issued < total; ++issued) issue((int)issued);
  while (done < total) {
    const int slot = done % stages;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P;}"
                   : "=r"(ok) : "r"(smem_u32(&bars[w][slot])), "r"(phase[slot]) : "memory");
    phase[slot] ^= 1;
    ++done;
    if (issued < total) { issue(slot); ++issued; }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t l2_bytes = 48ull << 20, hbm_bytes = 4ull << 30;
  char* buf;
  cudaMalloc(&buf, hbm_bytes);
  cudaMemset(buf, 1, hbm_bytes);
  int4* sink;
  cudaMalloc(&sink, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  // LDG, L2-resident
  for (int bpsm : {2, 4, 8}) {
    int iters = 20;
    ldg_kernel<<<sms * bpsm, 256>>>((int4*)buf, l2_bytes / 16, 2, sink);
    cudaEventRecord(a);
    ldg_kernel<<<sms * bpsm, 256>>>((int4*)buf, l2_bytes / 16, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG.128 L2-resident %d MB, %d CTA/SM: %.0f GB/s\n", (int)(l2_bytes >> 20), bpsm,
           l2_bytes * (double)iters / ms / 1e6);
  }
  // LDG, HBM
  ldg_kernel<<<sms * 4, 256>>>((int4*)buf, hbm_bytes / 16, 1, sink);
  cudaEventRecord(a);
  ldg_kernel<<<sms * 4, 256>>>((int4*)buf, hbm_bytes / 16, 2, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("LDG.128 HBM 4 GB: %.0f GB/s\n", hbm_bytes * 2.0 / ms / 1e6);
  // bulk copies, L2-resident: request size x in-flight depth x CTAs per SM
  struct Cfg { int chunk, stages, cta_per_sm; };
  Cfg cfgs[] = {{8192, 4, 1}, {8192, 4, 2}, {8192, 4, 4}, {8192, 8, 2}, {16384, 4, 2}, {16384, 3, 4},
                {32768, 3, 2}, {65536, 3, 1}, {4096, 8, 4}, {2048, 8, 8}};
  for (auto c : cfgs) {
    int smem = c.chunk * c.stages;
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int iters = 20, grid = sms * c.cta_per_sm;
    bulk_kernel<<<grid, 32, smem>>>(buf, l2_bytes, c.chunk, c.stages, 2);
    cudaEventRecord(a);
    bulk_kernel<<<grid, 32, smem>>>(buf, l2_bytes, c.chunk, c.stages, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaError_t e = cudaGetLastError();
    cudaEventElapsedTime(&ms, a, b);
    printf("cp.async.bulk chunk %6d x %d stages, %d CTA/SM: %6.0f GB/s %s\n", c.chunk, c.stages,
           c.cta_per_sm, l2_bytes * (double)iters / ms / 1e6, e ? cudaGetErrorString(e) : "");
  }
  struct MCfg { int chunk, stages, warps; };
  MCfg mc[] = {{8192, 3, 1}, {8192, 3, 2}, {8192, 3, 4}, {8192, 3, 8}, {16384, 2, 4}, {4096, 4, 8}};
  for (auto c : mc) {
    int smem = c.chunk * c.stages * c.warps;
    cudaFuncSetAttribute(bulk_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int iters = 20;
    bulk_multi_kernel<<<sms, 32 * c.warps, smem>>>(buf, l2_bytes, c.chunk, c.stages, 2);
    cudaEventRecord(a);
    bulk_multi_kernel<<<sms, 32 * c.warps, smem>>>(buf, l2_bytes, c.chunk, c.stages, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaError_t e = cudaGetLastError();
    cudaEventElapsedTime(&ms, a, b);
    printf("bulk multi-warp chunk %6d x %d stages x %d warps, 1 CTA/SM: %6.0f GB/s %s\n", c.chunk,
           c.stages, c.warps, l2_bytes * (double)iters / ms / 1e6, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
