// ptx.cuh — thin inline-PTX wrappers for the sm_100a features the kernels use:
// mbarrier, TMA (tiled + im2col), tcgen05 (TMEM alloc, MMA, commit, ld) and
// the UMMA shared-memory / instruction descriptors.
//
// Encodings follow the PTX ISA for sm_100a (descriptor bit layout as in
// CUTLASS's cute/arch/mma_sm100_desc.hpp, used here for reference only).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace tb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Explicit shared-space accesses (pointers derived through uintptr_t arithmetic
// lose their address space, and generic loads there cost hundreds of cycles).
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v));
}

// Materialise a value in a register at this point of the program (the empty
// volatile asm may not be moved across other volatile asm, e.g. griddepcontrol.wait):
// kernel parameters read after a PDL wait can miss the constant cache (~0.4 us each on
// the critical path, tools/cta_timeline.py), so producers pin the ones they need before it.
__device__ __forceinline__ int pin(int v) {
  asm volatile("" : "+r"(v));
  return v;
}

__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- debug timeline

// %globaltimer (ns) of kernel milestones of CTA b < 256 at
// trace[8192 + 8 * b + event] — only when a trace buffer is set
// (tir_b200_debug_set_trace; tools/floor_timeline.py). Null in production.
enum TraceEvent { TR_ENTRY = 0, TR_PDL_DONE = 1, TR_FIRST_FULL = 2, TR_FIRST_TFULL = 3, TR_STORES_DONE = 4,
                  TR_EXIT = 5, TR_FIRST_ISSUE = 6, TR_PRELOOP = 7 };
__device__ __forceinline__ void trace_event(unsigned long long* trace, int ev) {
  if (trace && blockIdx.x < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    trace[8192 + 8 * blockIdx.x + ev] = t;
  }
}

// Extra milestones j < 8 of CTA b < 256 at trace[10240 + 8 * b + j] (split-K combine
// timeline: tools/cta_timeline.py "x0".."x7"). Null in production.
__device__ __forceinline__ void trace_x(unsigned long long* trace, int j) {
  if (trace && blockIdx.x < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    trace[10240 + 8 * blockIdx.x + j] = t;
  }
}

// ---------------------------------------------------------------- mbarrier

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// Same, backing off with __nanosleep between polls: for waiters off the MMA
// issue path, whose spinning try_waits would otherwise share the MIO queue with
// the tcgen05.mma issue.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, uint32_t ns) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try_wait(addr, parity)) {
    __nanosleep(ns);
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > (1ull << 31)) __trap();
  }
}

// Bounded wait: a pipeline bug must surface as a trapped kernel (an error the
// host sees), never as a hung GPU. ~2^31 ns budget via %globaltimer.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try_wait(addr, parity)) {
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > (1ull << 31)) __trap();
  }
}

// ---------------------------------------------------------------- TMA

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}

// L2 prefetches of TMA boxes (no shared memory, no barrier). Issued BEFORE
// griddepcontrol.wait for a kernel's first loads: L2 is the point of coherence
// for global memory, so a line prefetched while the preceding kernel still
// writes it is updated in place by those writes — the prefetch only moves the
// DRAM latency of the first tile under the previous kernel's tail, it never
// lets stale data through (the real loads still come after the wait).
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* m, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(m), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* m, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(m), "r"(c0),
               "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// ---- TMA stores (smem -> global), bulk-group completion
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m),
      "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, const void* src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(m),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// Y += smem (element-wise fp32 add performed by the TMA unit).
__device__ __forceinline__ void tma_reduce_add_4d(const CUtensorMap* m, const void* src, int c0,
                                                  int c1, int c2, int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(m),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_store_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Wait until at most N committed bulk groups are still reading their smem source.
template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Programmatic dependent launch: wait for the preceding grid's memory, and let
// the next grid start launching (its CTAs fill SMs as ours exit).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// L2 prefetches of im2col boxes (same coordinates / offsets as the loads below).
__device__ __forceinline__ void tma_prefetch_im2col_3d(const CUtensorMap* m, int c, int w, int n, uint16_t ow) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.im2col [%0, {%1, %2, %3}], {%4};" ::"l"(m), "r"(c),
               "r"(w), "r"(n), "h"(ow)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_im2col_4d(const CUtensorMap* m, int c, int w, int h, int n,
                                                       uint16_t ow, uint16_t oh) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.im2col [%0, {%1, %2, %3, %4}], {%5, %6};" ::"l"(m),
               "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_im2col_5d(const CUtensorMap* m, int c, int w, int h, int d, int n,
                                                       uint16_t ow, uint16_t oh, uint16_t od) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.im2col [%0, {%1, %2, %3, %4, %5}], {%6, %7, %8};" ::"l"(
                   m),
               "r"(c), "r"(w), "r"(h), "r"(d), "r"(n), "h"(ow), "h"(oh), "h"(od)
               : "memory");
}

// im2col loads: coordinates (c, w[, h[, d]], n), offsets (w[, h[, d]]).
__device__ __forceinline__ void tma_im2col_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c,
                                              int w, int n, uint16_t ow) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2], {%6};" ::"r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(n), "h"(ow)
      : "memory");
}

__device__ __forceinline__ void tma_im2col_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c,
                                              int w, int h, int n, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}

__device__ __forceinline__ void tma_im2col_5d(void* dst, const CUtensorMap* m, uint64_t* bar, int c,
                                              int w, int h, int d, int n, uint16_t ow, uint16_t oh,
                                              uint16_t od) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], {%8, %9, %10};" ::"r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(d), "r"(n), "h"(ow), "h"(oh),
      "h"(od)
      : "memory");
}

// ---------------------------------------------------------------- tcgen05

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}

__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem], kind::f16 (fp16 inputs, fp32 accumulation).
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrives on `bar` once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets row
// (lane base + t), columns [col, col+32).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// 16 lanes x 256 bits, repeated 4x along columns (32 columns). Measured layout
// (tools/umma_probe.cu): thread t holds lane t/4 in r[4j], r[4j+1] and lane
// t/4 + 8 in r[4j+2], r[4j+3], columns 8j + 2(t%4) + {0, 1}: four consecutive
// threads own one 32-byte row segment.
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_16x256b_x2(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- fused epilogue

// v + bias[col], then max(v, 0) exactly as the reference's max(x, 0.0)
// (std::max: (v < 0) ? 0 : v, so NaN and -0.0 pass through like the interpreter).
// erf-form GELU, 0.5 v (1 + erf(v / sqrt 2)), with erf from Abramowitz & Stegun
// 7.1.26 (|error| <= 1.5e-7, below the fp16 output's half-ulp): branch-free,
// one exp2 and one reciprocal on the SFU plus 8 FMAs, so an unrolled epilogue
// chunk keeps 32 independent chains in flight (libm erff's branches serialise
// the single epilogue warp per sub-partition: BERT's FFN1 ran at 42% of the
// plain GEMM's rate with it).
__device__ __forceinline__ float gelu_erf(float v) {
  const float z = fabsf(v) * 0.70710678118654752f;
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.0f)));
  float poly = fmaf(t, 1.061405429f, -1.453152027f);
  poly = fmaf(t, poly, 1.421413741f);
  poly = fmaf(t, poly, -0.284496736f);
  poly = fmaf(t, poly, 0.254829592f);
  poly *= t;
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-z * z * 1.4426950408889634f));
  const float erf_abs = fmaf(-poly, e, 1.0f);
  const float erf = copysignf(erf_abs, v);
  return 0.5f * v * (1.0f + erf);
}

// act: 1 ReLU, 2 ReLU6, 3 GELU (erf form, BERT); 0 none. ReLU is the reference's
// max(x, 0.0) (std::max: (v < 0) ? 0 : v, so NaN and -0.0 pass through).
__device__ __forceinline__ float epi_act(float v, int act) {
  if (act == 1) return (v < 0.0f) ? 0.0f : v;
  if (act == 2) {
    v = (v < 0.0f) ? 0.0f : v;  // two flat selects: the nested ternary compiled
    return (v > 6.0f) ? 6.0f : v;  // to a divergent branch per element
  }
  if (act == 3) return gelu_erf(v);
  return v;
}

// In-place activation of N values; the branch on `act` is warp-uniform and sits
// outside the element loop so the loop body is straight-line code.
template <int N>
__device__ __forceinline__ void epi_act_n(float* v, int act) {
  if (act == 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = (v[i] < 0.0f) ? 0.0f : v[i];
  } else if (act == 2) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const float a = (v[i] < 0.0f) ? 0.0f : v[i];
      v[i] = (a > 6.0f) ? 6.0f : a;
    }
  } else if (act == 3) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = gelu_erf(v[i]);
  }
}

// Fused epilogue on N consecutive columns [col, col + N) of one output row, in
// the C-ABI order: v + bias[col + i], + residual[i], act. `lim` columns are
// valid (the rest lie past a group / tensor edge: never loaded, never stored by
// the caller). Bias and residual are fetched with 16-byte loads when the whole
// run is valid and aligned, so an epilogue chunk issues a handful of independent
// loads instead of N dependent ones.
template <int N>
__device__ __forceinline__ void epi_run(float* v, const float* bias, int64_t col, int lim,
                                        const uint16_t* res, int act) {
  if (bias) {
    const float* b = bias + col;
    if (N % 4 == 0 && lim >= N && (reinterpret_cast<uintptr_t>(b) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < N; i += 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(b + i));
        v[i] += t.x; v[i + 1] += t.y; v[i + 2] += t.z; v[i + 3] += t.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i)
        if (i < lim) v[i] += __ldg(b + i);
    }
  }
  if (res) {
    if (N % 8 == 0 && lim >= N && (reinterpret_cast<uintptr_t>(res) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < N; i += 8) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(res + i));
        const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __half22float2(h[j]);
          v[i + 2 * j] += f.x;
          v[i + 2 * j + 1] += f.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i)
        if (i < lim)
          v[i] += __half2float(__ushort_as_half(__ldg(reinterpret_cast<const unsigned short*>(res) + i)));
    }
  }
  epi_act_n<N>(v, act);
}

// ---------------------------------------------------------------- descriptors

// UMMA shared-memory matrix descriptor (sm_100: version field = 1).
//   layout: 0 = no swizzle (interleave), 2 = 128B, 4 = 64B, 6 = 32B swizzle.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  d |= static_cast<uint64_t>(layout & 7u) << 61;
  return d;
}

// Instruction descriptor, kind::f16: A,B fp16, D fp32.
//   a_mn_major / b_mn_major: 0 = K-major, 1 = MN-major.
__host__ __device__ constexpr uint32_t idesc_f16_f32(uint32_t M, uint32_t N, uint32_t a_mn_major,
                                                     uint32_t b_mn_major) {
  return (1u << 4)                   // D format: F32
         | (0u << 7) | (0u << 10)    // A, B format: F16
         | (a_mn_major << 15) | (b_mn_major << 16)
         | ((N >> 3) << 17)          // N / 8
         | ((M >> 4) << 24);         // M / 16
}

}  // namespace tb
