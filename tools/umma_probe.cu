// umma_probe.cu — hardware probe: can a K-major SWIZZLE_128B UMMA descriptor
// start at an arbitrary 128-byte row of a TMA-written (swizzled) tile, and is
// the descriptor's base_offset field needed? Computes D = A[o:o+128, :64] x I
// for several row offsets o and reports whether D reproduces A's rows.
// Not part of the product (design probe for the halo convolution kernel).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2207_04296_b200/csrc/ptx.cuh"

using namespace tb;

__global__ void probe(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      float* out, int row_off, int use_base_offset) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;              // 256 rows x 128 B
  uint8_t* sB = smem + 256 * 128;  // 64 rows (K) x 64 cols (N) MN-major, 8 KB
  __shared__ __align__(8) uint64_t bar, mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  if (warp == 0) { tmem_alloc(&tslot, 64); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 256 * 128 + 64 * 128);
    tma_load_2d(sA, &mapA, &bar, 0, 0);
    tma_load_2d(sA + 128 * 128, &mapA, &bar, 0, 128);
    tma_load_2d(sB, &mapB, &bar, 0, 0);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sA) + (row_off < 0 ? 0 : row_off) * 128;
    uint64_t ad = smem_desc(a, 16, 1024, 2);
    if (use_base_offset) ad |= (uint64_t)((a >> 7) & 7) << 49;
    const uint64_t bd0 = smem_desc(smem_u32(sB), 8192, 1024, 2);
    const uint32_t idesc = idesc_f16_f32(128, 64, 0, 1);
    for (int k = 0; k < 4; ++k) umma_f16(tmem, ad + ((32 * k) >> 4), bd0 + ((16 * 128 * k) >> 4), idesc, k > 0);
    umma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  if (row_off < 0) {  // layout probe for tcgen05.ld.16x256b.x1 (warp 0, lanes 0..15)
    if (warp == 0) {
      uint32_t a0, a1, a2, a3;
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(tmem));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      out[lane * 4 + 0] = __uint_as_float(a0);
      out[lane * 4 + 1] = __uint_as_float(a1);
      out[lane * 4 + 2] = __uint_as_float(a2);
      out[lane * 4 + 3] = __uint_as_float(a3);
    }
  } else if (warp < 4) {
    uint32_t r[32];
    for (int c0 = 0; c0 < 64; c0 += 32) {
      tmem_ld_32x32b_x32(tmem + ((warp * 32u) << 16) + c0, r);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) out[(warp * 32 + lane) * 64 + c0 + i] = __uint_as_float(r[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 64);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  // A: 256 x 64 with A[r][c] = r + c/64 (distinct per row), B = identity (K x N)
  __half hA[256 * 64], hB[64 * 64];
  for (int r = 0; r < 256; ++r)
    for (int c = 0; c < 64; ++c) hA[r * 64 + c] = __float2half((float)((r * 7 + c) % 512) - 256.0f);
  for (int k = 0; k < 64; ++k)
    for (int n = 0; n < 64; ++n) hB[k * 64 + n] = __float2half(k == n ? 1.0f : 0.0f);
  void *dA, *dB;
  float* dO;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  CUtensorMap mA, mB;
  cuuint64_t dimsA[2] = {64, 256}, strA[1] = {128};
  cuuint32_t boxA[2] = {64, 128}, es[2] = {1, 1};
  enc(&mA, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dA, dimsA, strA, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t dimsB[2] = {64, 64}, strB[1] = {128};
  cuuint32_t boxB[2] = {64, 64};
  enc(&mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dB, dimsB, strB, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  static float hO[128 * 64];
  for (int use_bo = 0; use_bo < 2; ++use_bo) {
    for (int off : {0, 1, 2, 3, 5, 8, 9, 13, 58, 59, 116, 118}) {
      probe<<<1, 128, 64 * 1024>>>(mA, mB, dO, off, use_bo);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("off %d: %s\n", off, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int r = 0; r < 128; ++r)
        for (int c = 0; c < 64; ++c)
          if (hO[r * 64 + c] != __half2float(hA[(r + off) * 64 + c])) ++bad;
      printf("base_offset=%d row_off=%3d : %s (%d mismatches)\n", use_bo, off, bad ? "WRONG" : "exact", bad);
    }
  }
  // 16x256b layout: D = A[0:128] x I. Run twice: A = row index, then A = column index.
  int rowid[128], colid[128];
  for (int pass = 0; pass < 2; ++pass) {
    for (int r = 0; r < 256; ++r)
      for (int c = 0; c < 64; ++c) hA[r * 64 + c] = __float2half((float)(pass == 0 ? r : c));
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    probe<<<1, 128, 64 * 1024>>>(mA, mB, dO, -1, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(hO, dO, 128 * 4, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 128; ++i) (pass == 0 ? rowid : colid)[i] = (int)hO[i];
  }
  for (int t = 0; t < 32; ++t) {
    printf("16x256b thread %2d:", t);
    for (int j = 0; j < 4; ++j) printf(" r%d=(lane %d, col %d)", j, rowid[t * 4 + j], colid[t * 4 + j]);
    printf("\n");
  }
  return 0;
}
