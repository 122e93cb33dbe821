// tmabw.cu — microbenchmark: tensor-mode TMA (cp.async.bulk.tensor.2d) load
// throughput from an L2-resident fp16 matrix, by box shape / swizzle / number
// of issuing warps / CTAs per SM. Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmabw tools/tmabw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct Args {
  int box_cols, box_rows, tiles_c, tiles_r, stages, iters;
};

// Each issuing warp (lane 0) runs its own ring of `stages` slots.
__global__ void tma_kernel(const __grid_constant__ CUtensorMap map, Args a) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = (char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[8][8];
  const int w = threadIdx.x / 32, nw = blockDim.x / 32;
  const int bytes = a.box_cols * a.box_rows * 2;
  if (threadIdx.x % 32 == 0) {
    for (int i = 0; i < a.stages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[w][i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x % 32 != 0) return;
  char* my = smem + (size_t)w * a.stages * bytes;
  const int ntiles = a.tiles_c * a.tiles_r;
  const int gid = blockIdx.x * nw + w, gstride = gridDim.x * nw;
  uint32_t phase[8] = {0};
  long total = (long)a.iters * ((ntiles + gstride - 1 - gid) / gstride), issued = 0, done = 0;
  int next = gid;
  auto issue = [&](int slot) {
    int t = next % ntiles;
    next += gstride;
    int c0 = (t % a.tiles_c) * a.box_cols, r0 = (t / a.tiles_c) * a.box_rows;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[w][slot])),
                 "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(my + (size_t)slot * bytes)),
        "l"(&map), "r"(smem_u32(&bars[w][slot])), "r"(c0), "r"(r0) : "memory");
  };
  for (; issued < a.stages && issued < total; ++issued) issue((int)issued);
  while (done < total) {
    const int slot = done % a.stages;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P;}"
                   : "=r"(ok) : "r"(smem_u32(&bars[w][slot])), "r"(phase[slot]) : "memory");
    phase[slot] ^= 1;
    ++done;
    if (issued < total) { issue(slot); ++issued; }
  }
}

// im2col variant: 4-D NHWC, 128 pixels x C channels per request.
struct Im2colArgs { int n, h, w, pix_tiles, cblocks, box_ch, stages, iters; };
__global__ void im2col_kernel(const __grid_constant__ CUtensorMap map, Im2colArgs a) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = (char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[8][8];
  const int w = threadIdx.x / 32, nw = blockDim.x / 32;
  const int bytes = 128 * a.box_ch * 2;
  if (threadIdx.x % 32 == 0) {
    for (int i = 0; i < a.stages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[w][i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x % 32 != 0) return;
  char* my = smem + (size_t)w * a.stages * bytes;
  const int ntiles = a.pix_tiles * a.cblocks * 9;
  const int gid = blockIdx.x * nw + w, gstride = gridDim.x * nw;
  uint32_t phase[8] = {0};
  long total = (long)a.iters * ((ntiles + gstride - 1 - gid) / gstride), issued = 0, done = 0;
  int next = gid;
  auto issue = [&](int slot) {
    int t = next % ntiles;
    next += gstride;
    int tap = t % 9, rest = t / 9;
    int cb = rest % a.cblocks, pt = rest / a.cblocks;
    int m0 = pt * 128;
    int x = m0 % a.w, y = (m0 / a.w) % a.h, n = m0 / (a.w * a.h);
    uint16_t ox = tap % 3, oy = tap / 3;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[w][slot])),
                 "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(my + (size_t)slot * bytes)),
        "l"(&map), "r"(smem_u32(&bars[w][slot])), "r"(cb * a.box_ch), "r"(x - 1), "r"(y - 1), "r"(n),
        "h"(ox), "h"(oy) : "memory");
  };
  for (; issued < a.stages && issued < total; ++issued) issue((int)issued);
  while (done < total) {
    const int slot = done % a.stages;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P;}"
                   : "=r"(ok) : "r"(smem_u32(&bars[w][slot])), "r"(phase[slot]) : "memory");
    phase[slot] ^= 1;
    ++done;
    if (issued < total) { issue(slot); ++issued; }
  }
}

using Im2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  const int cols = 4096, rows = 6144;  // 48 MB fp16, L2-resident
  void* buf;
  cudaMalloc(&buf, (size_t)cols * rows * 2);
  cudaMemset(buf, 0, (size_t)cols * rows * 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int bc, br, swz, warps, cta_per_sm, stages; const char* name; };
  Cfg cfgs[] = {
      {64, 128, 128, 1, 1, 4, "sw128 64x128 (16KB) 1 warp"},
      {64, 128, 128, 2, 1, 4, "sw128 64x128 (16KB) 2 warps"},
      {64, 128, 128, 4, 1, 3, "sw128 64x128 (16KB) 4 warps"},
      {64, 128, 128, 1, 2, 4, "sw128 64x128 (16KB) 1 warp x 2 CTA/SM"},
      {64, 128, 128, 1, 4, 3, "sw128 64x128 (16KB) 1 warp x 4 CTA/SM"},
      {64, 256, 128, 1, 1, 4, "sw128 64x256 (32KB) 1 warp"},
      {64, 256, 128, 2, 1, 3, "sw128 64x256 (32KB) 2 warps"},
      {64, 64, 128, 4, 1, 4, "sw128 64x64 (8KB) 4 warps"},
      {256, 64, 0, 1, 1, 4, "noswz 256x64 (32KB, 512B rows) 1 warp"},
      {256, 64, 0, 2, 1, 3, "noswz 256x64 (32KB, 512B rows) 2 warps"},
      {64, 128, 0, 1, 1, 4, "noswz 64x128 (16KB, 128B rows) 1 warp"},
      {32, 256, 64, 1, 1, 4, "sw64 32x256 (16KB, 64B rows) 1 warp"},
  };
  for (auto c : cfgs) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)c.bc, (cuuint32_t)c.br};
    cuuint32_t es[2] = {1, 1};
    CUtensorMapSwizzle sw = c.swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : c.swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                          : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", c.name, (int)r); continue; }
    Args a{c.bc, c.br, cols / c.bc, rows / c.br, c.stages, 10};
    int bytes = c.bc * c.br * 2;
    int smem = bytes * c.stages * c.warps + 1024;
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int grid = sms * c.cta_per_sm;
    tma_kernel<<<grid, 32 * c.warps, smem>>>(map, Args{a.box_cols, a.box_rows, a.tiles_c, a.tiles_r, a.stages, 1});
    cudaEventRecord(e0);
    tma_kernel<<<grid, 32 * c.warps, smem>>>(map, a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaError_t err = cudaGetLastError();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double total = (double)cols * rows * 2 * a.iters;
    printf("%-44s %6.0f GB/s  (%.1f B/clk/SM @1.87GHz) %s\n", c.name, total / ms / 1e6,
           total / ms / 1e6 / sms / 1.87, err ? cudaGetErrorString(err) : "");
  }
  // im2col: N16 56x56 C64 (6.4 MB, L2-resident), 3x3 taps, pad 1
  void* fn2 = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn2, cudaEnableDefault, &q);
  Im2colFn enc2 = (Im2colFn)fn2;
  for (int box_ch : {64, 32}) {
    for (int warps : {1, 2, 4}) {
      const int N = 16, H = 56, W = 56, C = 64;
      CUtensorMap map;
      cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
      cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
      int lo[2] = {-1, -1}, up[2] = {-1, -1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = enc2(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, buf, dims, strides, lo, up, box_ch, 128, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        box_ch == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("im2col encode failed %d\n", (int)r); continue; }
      Im2colArgs a{N, H, W, N * H * W / 128, C / box_ch, box_ch, 3, 10};
      int bytes = 128 * box_ch * 2;
      int smem = bytes * a.stages * warps + 1024;
      cudaFuncSetAttribute(im2col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      Im2colArgs a1 = a; a1.iters = 1;
      im2col_kernel<<<sms, 32 * warps, smem>>>(map, a1);
      cudaEventRecord(e0);
      im2col_kernel<<<sms, 32 * warps, smem>>>(map, a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaError_t err = cudaGetLastError();
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double total = (double)a.pix_tiles * a.cblocks * 9 * bytes * a.iters;
      printf("im2col 4D box %d ch x 128 px, %d warps           %6.0f GB/s  (%.1f B/clk/SM) %s\n", box_ch,
             warps, total / ms / 1e6, total / ms / 1e6 / sms / 1.87, err ? cudaGetErrorString(err) : "");
    }
  }
  return 0;
}
