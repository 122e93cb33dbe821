// rowpack.cuh — small-channel convolution (CI = 3 stems: the C3D paper shape,
// 7x7 / 3x3 stride-2 stems) with the MMA's A operand packed into TENSOR memory.
//
// Why: with CI = 3 a 7x7 tap row carries 21 useful values. im2col pieces of
// (kw, c) (the igemm path) stream each input pixel ~KH*KD times through L2 into
// shared memory and need a 411 MB relayout for the C3D paper shape; the MMA then
// re-reads every A row from shared memory (SS mode: 48 cycles per 128x64x16 MMA,
// tools/mma_rate2.cu). Here:
//   * the producer TMA-loads RAW input rows: for one output tile (R rows x Wt
//     columns) and one input depth plane, the box of box_h input rows x box_w
//     elements of the [W*CI] row (4.7 KB for C3D) — zero fill is the padding;
//   * 8 builder warps turn it into the packed A operand directly in TMEM: TMEM
//     lane m = output pixel (m / Wt, m % Wt); its K vector is the kh taps of the
//     plane back to back, each tap the KW*CI elements of input row sh*r + dh*kh
//     from element sw*CI*c on (KW runs of CI contiguous elements, dw*CI apart:
//     32-bit shared loads and one byte permute per word), padded to an even
//     count (WPK 32-bit words);
//     tcgen05.st writes them (measured 605 B/clk);
//   * the MMA warp issues kind::f16 MMAs with A in TMEM (TS mode, 32 cycles per
//     128x64x16 — the full tensor rate) and B = the packed weight panel, resident
//     in shared memory for the whole kernel ([KD][Kp][CO], Kp = 16*ksteps rows
//     laid out like the TMEM K vector);
//   * a work unit is (image, group of 2 output depths, tile): each input plane is
//     loaded and packed once and feeds both output depths' accumulators (with
//     their own kd), double-buffered accumulators let the TMA-store epilogue of
//     unit i overlap the MMAs of unit i+1.
// Reduction order: (kd, kh, kw, c) per output, exactly the reference's loop nest
// order reassociated inside the tensor core; on the reference input distribution
// every partial sum is exact (bit-identical results, tests/test_gpu_parity.py).
#pragma once

#include "ptx.cuh"

namespace tb {

constexpr int kRpProducers = 4;   // TMA producer warps (raw boxes of planes it = pw mod 4)
constexpr int kRpThreads = 544;  // warps 0-3 epilogue, 4-11 builders, 12 MMA, 13-16 producers
constexpr int kRpMmaWarp = 12;   // on SM sub-partition 0 (warp % 4 == 0)
constexpr int kRpMaxSlots = 5;   // TMEM accumulator ring (p.nacc slots): output depths in flight + one draining
constexpr int kRpMaxA = 4;       // TMEM A-buffer ring (p.nabuf buffers of KWORDS columns after the accumulators)
constexpr int kRpDescRing = 16;  // plane descriptors in flight (> raw stages + A buffers: no reuse race)

struct alignas(64) RowpackParams {
  CUtensorMap tmX;  // 3-D over X[N*D, H, W*CI] fp16: box {box_w, box_h, 1}, no swizzle
  CUtensorMap tmB;  // 2-D over Bp[KD*Kp, CO] fp16: box {BN, Kp}, SW128 (BN 64) / SW64 (BN 32)
  CUtensorMap tmY;  // 4-D over Y[N*OD, OH, OW, CO]: box {32, Wt, R, 1}
  int32_t n, d, ci;
  int32_t od, oh, ow;
  int32_t kd, sd, sh, sw, pd, ph, pw, dd, dh;
  int32_t R, Wt, tiles_h, tiles_w, total_units;
  int32_t kp;  // packed K rows per kd (16 * ksteps)
  int32_t box_w, box_h;
  int32_t shift;  // elements between the box's 16-byte-aligned start column and the tile's first input element
  int32_t stages, slot_bytes;
  int32_t out_f16, store_mode;  // store_mode 1: TMA store, 2: TMA reduce-add (Y += conv)
  int32_t stage_bytes;
  const float* bias;  // fused epilogue (nullable): per-output-channel bias, then activation `act`
  int32_t act;        // 0 none, 1 ReLU, 2 ReLU6, 3 GELU (epi_act)
  int32_t backoff_ns, backoff_ns2;  // poll back-off of producers / epilogue, and of the builders
  int32_t debug;  // timing experiments only (wrong results): 1 builders skip the raw loads, 2 no output
                  // stores, 4 no A build at all, 16 no raw loads
  unsigned long long* trace;
};

// tcgen05.st.32x32b of N consecutive columns (lane = thread's TMEM lane).
template <int N>
__device__ __forceinline__ void tmem_st_n(uint32_t taddr, const uint32_t* v);
template <>
__device__ __forceinline__ void tmem_st_n<1>(uint32_t t, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t), "r"(v[0]));
}
template <>
__device__ __forceinline__ void tmem_st_n<2>(uint32_t t, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(t), "r"(v[0]), "r"(v[1]));
}
template <>
__device__ __forceinline__ void tmem_st_n<4>(uint32_t t, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(t), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]));
}
template <>
__device__ __forceinline__ void tmem_st_n<8>(uint32_t t, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(t),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
template <>
__device__ __forceinline__ void tmem_st_n<16>(uint32_t t, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(t),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
template <>
__device__ __forceinline__ void tmem_st_n<32>(uint32_t t, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(t),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}

// N columns as a compile-time sequence of power-of-two stores.
template <int N>
__device__ __forceinline__ void tmem_st_words(uint32_t t, const uint32_t* v) {
  if constexpr (N >= 32) {
    tmem_st_n<32>(t, v);
    tmem_st_words<N - 32>(t + 32, v + 32);
  } else if constexpr (N >= 16) {
    tmem_st_n<16>(t, v);
    tmem_st_words<N - 16>(t + 16, v + 16);
  } else if constexpr (N >= 8) {
    tmem_st_n<8>(t, v);
    tmem_st_words<N - 8>(t + 8, v + 8);
  } else if constexpr (N >= 4) {
    tmem_st_n<4>(t, v);
    tmem_st_words<N - 4>(t + 4, v + 4);
  } else if constexpr (N >= 2) {
    tmem_st_n<2>(t, v);
    tmem_st_words<N - 2>(t + 2, v + 2);
  } else if constexpr (N == 1) {
    tmem_st_n<1>(t, v);
  }
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

template <int BN>
struct RowpackCfg {
  static constexpr int kBRowBytes = BN * 2;
  static constexpr uint32_t kBLayout = kBRowBytes == 128 ? 2u : 4u;  // SW128 / SW64
  static constexpr uint32_t kIdesc = idesc_f16_f32(128, BN, 0, 1);
};

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// One tap's (kw, c) window: KW runs of CI contiguous elements, DW*CI elements
// apart (dilation DW), packed as KW*CI elements padded to an even count (WPK
// 32-bit words). Element k of the window sits kOff(k) elements past the run start.
template <int KW, int CI, int DW>
struct TapWindow {
  static constexpr int kKwc = KW * CI;
  static constexpr int kWpk = (kKwc + 1) / 2;
  static constexpr int kSpan = (KW - 1) * DW * CI + CI;  // elements from the first to past the last
  __host__ __device__ static constexpr int off(int k) { return (k / CI) * DW * CI + k % CI; }
};

// Columns [C0, C1) of one lane's TMEM K vector, stored in 8-column tcgen05.st
// chunks at 8-aligned columns. Column k is word k % WPK of tap k / WPK: the
// window elements 2j, 2j+1 (j = k % WPK) of raw row e0 + tap*tap_step. Every run
// of a kernel starts at the same element parity (ODD): the aligned words spanning
// the window are loaded once per tap and each output word is one byte permute of
// two of them (compile-time selectors). Columns past KH*WPK are the K padding,
// an odd KW*CI pads each tap with one zero. Lanes past the tile's pixels
// (r = c = 0) build a copy of pixel 0: their TMEM rows only feed discarded rows.
template <int C0, int C1, int KH, int KW, int CI, int DW, bool ODD>
__device__ __forceinline__ void build_cols(uint32_t src, uint32_t e0, uint32_t tap_step, uint32_t abase) {
  using Win = TapWindow<KW, CI, DW>;
  constexpr int WPK = Win::kWpk;
  constexpr int kN = C1 - C0;
  constexpr int kT0 = C0 / WPK;
  constexpr int kT1 = ((C1 - 1) / WPK < KH - 1) ? (C1 - 1) / WPK : KH - 1;
  constexpr int kNW = (Win::kSpan + (ODD ? 1 : 0) + 1) / 2;  // aligned words covering the window
  uint32_t w[kN];
#pragma unroll
  for (int i = 0; i < kN; ++i) w[i] = 0u;
#pragma unroll
  for (int t = kT0; t <= kT1; ++t) {
    const uint32_t a = src + (((e0 + static_cast<uint32_t>(t) * tap_step) >> 1) << 2);
    uint32_t v[kNW];
#pragma unroll
    for (int j = 0; j < kNW; ++j) v[j] = lds_u32(a + 4 * j);
#pragma unroll
    for (int j = 0; j < WPK; ++j) {
      const int k = t * WPK + j;
      if (k >= C0 && k < C1) {
        const int h0 = Win::off(2 * j) + (ODD ? 1 : 0);  // half-word index of element 2j
        if (2 * j + 1 < Win::kKwc) {
          const int h1 = Win::off(2 * j + 1) + (ODD ? 1 : 0);
          const uint32_t lo_sel = (h0 & 1) ? 0x32u : 0x10u;
          const uint32_t hi_sel = (h1 / 2 == h0 / 2) ? ((h1 & 1) ? 0x32u : 0x10u) : ((h1 & 1) ? 0x76u : 0x54u);
          w[k - C0] = __byte_perm(v[h0 / 2], v[h1 / 2], lo_sel | (hi_sel << 8));
        } else {
          w[k - C0] = (h0 & 1) ? (v[h0 / 2] >> 16) : (v[h0 / 2] & 0xFFFFu);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kN; c += 8) tmem_st_n<8>(abase + C0 + c, w + c);
}

template <int BN, int KH, int KW, int CI, int DW, bool D3>
__global__ void __launch_bounds__(kRpThreads, 1) conv_rowpack_kernel(const __grid_constant__ RowpackParams p) {
  using Cfg = RowpackCfg<BN>;
  constexpr int WPK = TapWindow<KW, CI, DW>::kWpk;
  constexpr int kWords = (KH * WPK + 7) / 8 * 8;   // TMEM columns of one A buffer
  constexpr int kSteps = kWords / 8;               // K16 steps per plane
  constexpr int kHalfCols = (kSteps + 1) / 2 * 8;  // builder half 0: columns [0, kHalfCols), half 1: the rest
  // TMEM: nacc * BN accumulator columns, then nabuf A buffers. Compile-time, so the
  // per-plane / per-depth ring arithmetic is multiply-shift, not division: 3-D
  // convs keep ceil(KD/sd) <= 4 depths in flight + one draining, 2-D convs one
  // tile computing + one draining; the A ring takes what is left (<= 4).
  constexpr int nacc = D3 ? kRpMaxSlots : 2;
  constexpr int nabuf_fit = (512 - nacc * BN) / kWords;
  constexpr int nabuf = nabuf_fit < kRpMaxA ? nabuf_fit : kRpMaxA;
  static_assert(nabuf >= 2, "TMEM budget");
  constexpr uint32_t a_col = static_cast<uint32_t>(nacc * BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int S = p.stages;
  const int b_rows = p.kd * p.kp;
  uint8_t* sB = smem;
  uint8_t* epi = sB + static_cast<size_t>(b_rows) * Cfg::kBRowBytes;  // 1024-aligned (host)
  uint8_t* raw = epi + 2 * p.stage_bytes;
  uint64_t* rfull = reinterpret_cast<uint64_t*>(raw + static_cast<size_t>(S) * p.slot_bytes);
  uint64_t* rempty = rfull + S;
  uint64_t* afull = rempty + S;          // [kRpMaxA]
  uint64_t* afree = afull + kRpMaxA;     // [kRpMaxA]
  uint64_t* tfull = afree + kRpMaxA;     // [kRpMaxSlots]
  uint64_t* tempty = tfull + kRpMaxSlots;  // [kRpMaxSlots]
  uint64_t* bfull = tempty + kRpMaxSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  // per-plane MMA descriptors (kRpDescRing x 3 uint4), written by the producer that
  // loads the plane, read by the MMA thread after the plane's A buffer is published
  uint4* pdesc = reinterpret_cast<uint4*>((reinterpret_cast<uintptr_t>(tmem_slot + 1) + 15) & ~uintptr_t(15));

  if (threadIdx.x == 0) trace_event(p.trace, TR_ENTRY);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 32 * 13 + 1) {
    prefetch_tmap(&p.tmX);
    prefetch_tmap(&p.tmB);
    prefetch_tmap(&p.tmY);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&rfull[i], 1);
      mbar_init(&rempty[i], 8);  // the 8 builder warps
    }
    for (int i = 0; i < kRpMaxA; ++i) {
      mbar_init(&afull[i], 8);
      mbar_init(&afree[i], 1);
    }
    for (int i = 0; i < kRpMaxSlots; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);  // epilogue threads
    }
    mbar_init(bfull, 1);
    fence_barrier_init();
  }
  if (warp == kRpMmaWarp) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  // block 0's SM-clock trace (tools/cta_timeline.py): producer [2i], MMA [256 + 2i],
  // epilogue [512 + 2u], builder warp 4 [640 + 3i]
  unsigned long long* trace = (blockIdx.x == 0) ? p.trace : nullptr;
  if (trace && threadIdx.x == 0) trace[1023] = clock64();

  // A unit is one spatial tile (n, tile row, tile col) through the whole depth:
  // input planes di = lo .. hi in order; plane di feeds output depths
  // od in [od_first(di), od_last(di)] with kd = di - (od*sd - pd) (depth dilation 1).
  auto decompose = [&](int u, int& n, int& th, int& tw) {
    tw = u % p.tiles_w;
    const int r = u / p.tiles_w;
    th = r % p.tiles_h;
    n = r / p.tiles_h;
  };
  const int plane_lo = 0 > -p.pd ? 0 : -p.pd;  // first plane any output depth reads
  int plane_hi = (p.od - 1) * p.sd - p.pd + p.kd - 1;
  if (plane_hi > p.d - 1) plane_hi = p.d - 1;
  // (stride 1 / 2 divide by shifts; the general stride keeps the division)
  auto div_sd = [&](int x) { return p.sd == 1 ? x : p.sd == 2 ? (x >> 1) : x / p.sd; };  // x >= 0
  auto od_range = [&](int di, int& o0, int& o1) {
    const int t = di + p.pd - (p.kd - 1);  // od*sd >= t
    o0 = t <= 0 ? 0 : div_sd(t + p.sd - 1);
    o1 = div_sd(di + p.pd);
    if (o1 > p.od - 1) o1 = p.od - 1;
  };

  if (warp >= 13) {
    // ------------------------------------------------------------ producers
    // One raw box (box_h short rows) per plane; a TMA issue costs an issuing warp
    // ~1000+ cycles for such a box, so 4 producer warps take planes it = pw (mod 4).
    const int pw = static_cast<int>(warp) - 13;
    if (elect_one()) {
      pdl_wait();  // X / W may be produced by the preceding kernels
      if (pw == 0) {
        trace_event(p.trace, TR_PDL_DONE);
        if (static_cast<int>(blockIdx.x) < p.total_units) {
          // the packed weight panel, resident for the whole kernel: one box per kd
          mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(b_rows) * Cfg::kBRowBytes);
          for (int k = 0; k < p.kd; ++k)
            tma_load_2d(sB + static_cast<size_t>(k) * p.kp * Cfg::kBRowBytes, &p.tmB, bfull, 0, k * p.kp);
        }
      }
      int it = 0;
      int ubase_p = 0;
      const uint32_t kd_step_p = (static_cast<uint32_t>(p.kp) * Cfg::kBRowBytes) >> 4;
      for (int u = blockIdx.x; u < p.total_units; u += gridDim.x, ubase_p += p.od) {
        int n, th, tw;
        decompose(u, n, th, tw);
        // the box starts `shift` elements before the tile's first input element (16-byte aligned)
        const int x0 = (tw * p.Wt * p.sw - p.pw) * p.ci - p.shift;
        const int y0 = th * p.R * p.sh - p.ph;
        for (int di = plane_lo; di <= plane_hi; ++di) {
          int o0, o1;
          od_range(di, o0, o1);
          if (o0 > o1) continue;
          if ((it & (kRpProducers - 1)) == pw) {
            const uint32_t slot = static_cast<uint32_t>(it % S), phase = static_cast<uint32_t>(it / S) & 1u;
            mbar_wait_backoff(&rempty[slot], phase ^ 1, p.backoff_ns);
            if (trace && it < 128) trace[2 * it] = clock64();
            // the plane's MMA bookkeeping, off the MMA thread (released by the rfull arrive
            // below; the MMA thread reads it after acquiring the plane's afull); 2-D convs
            // have one plane per tile, which the MMA thread handles inline
            if constexpr (D3) {
              uint32_t w[12] = {static_cast<uint32_t>(o1 - o0 + 1), 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
              for (int i = 0; i < kRpMaxSlots - 1 && o0 + i <= o1; ++i) {
                const int od = o0 + i, g = ubase_p + od, base = od * p.sd - p.pd;
                const uint32_t first = di == (base > 0 ? base : 0);
                const uint32_t last = di == (base + p.kd - 1 < p.d - 1 ? base + p.kd - 1 : p.d - 1);
                w[1 + 2 * i] = static_cast<uint32_t>(di - base) * kd_step_p;
                w[2 + 2 * i] = static_cast<uint32_t>(g % nacc) | (first << 4) | (last << 5) |
                               ((static_cast<uint32_t>(g / nacc) & 1u) << 6);
              }
              uint4* dst = pdesc + (it % kRpDescRing) * 3;
              dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
              dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
              dst[2] = make_uint4(w[8], w[9], w[10], w[11]);
            }
            if (p.debug & 16) {
              mbar_arrive(&rfull[slot]);  // timing experiment: no raw load
            } else {
              mbar_arrive_expect_tx(&rfull[slot], static_cast<uint32_t>(p.box_w * p.box_h * 2));
              tma_load_3d(raw + static_cast<size_t>(slot) * p.slot_bytes, &p.tmX, &rfull[slot], x0, y0,
                          n * p.d + di);
            }
            if (trace && it < 128) trace[2 * it + 1] = clock64();
          }
          ++it;
        }
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ------------------------------------------------------------ builders
    // warp 4 + 4*half + q: TMEM lane quadrant q, K-vector columns of its half
    const int bw = static_cast<int>(warp) - 4;
    const int q = bw & 3, half = bw >> 2;
    const int m = q * 32 + static_cast<int>(lane);
    const bool live = m < p.R * p.Wt;
    const int r = live ? m / p.Wt : 0, c = live ? m % p.Wt : 0;  // dead lanes copy pixel 0
    // element offset of the lane's first tap run in the raw box (row sh*r, column
    // shift + sw*CI*c; tap kh adds dh*kh rows); tap_step is even (box_w % 8 == 0)
    const uint32_t e0 = static_cast<uint32_t>(r * p.sh) * static_cast<uint32_t>(p.box_w) +
                        static_cast<uint32_t>(p.shift + c * p.sw * p.ci);
    const uint32_t tap_step = static_cast<uint32_t>(p.dh) * static_cast<uint32_t>(p.box_w);
    const bool odd = (p.shift & 1) != 0;
    const uint32_t lane_base = tmem_base + ((static_cast<uint32_t>(q) * 32u) << 16) + a_col;
    const uint32_t raw_s = smem_u32(raw);
    uint32_t slot = 0, phase = 0;
    uint32_t pi = 0;  // plane counter (A buffer = pi % nabuf)
    for (int u = blockIdx.x; u < p.total_units; u += gridDim.x) {
      for (int di = plane_lo; di <= plane_hi; ++di) {
        int o0, o1;
        od_range(di, o0, o1);
        if (o0 > o1) continue;
        mbar_wait_backoff(&rfull[slot], phase, p.backoff_ns2);
        const bool tr = trace && warp == 4 && lane == 0 && pi < 64;
        if (tr) trace[640 + 3 * pi] = clock64();
        const uint32_t src = raw_s + slot * static_cast<uint32_t>(p.slot_bytes);
        const uint32_t ab = pi % nabuf, use = pi / nabuf;
        mbar_wait_backoff(&afree[ab], (use & 1) ^ 1, p.backoff_ns2);  // the MMAs of plane pi - nabuf are done with buffer ab
        tc_fence_after();
        if (tr) trace[641 + 3 * pi] = clock64();
        const uint32_t abase = lane_base + ab * kWords;
        if (p.debug & 4) {
          // timing experiment: no A build at all (stale TMEM)
        } else if (p.debug & 1) {
          uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          if (half == 0)
            for (int c0 = 0; c0 < kHalfCols; c0 += 8) tmem_st_n<8>(abase + c0, z);
          else
            for (int c0 = kHalfCols; c0 < kWords; c0 += 8) tmem_st_n<8>(abase + c0, z);
        } else if (half == 0) {
          if (odd) build_cols<0, kHalfCols, KH, KW, CI, DW, true>(src, e0, tap_step, abase);
          else build_cols<0, kHalfCols, KH, KW, CI, DW, false>(src, e0, tap_step, abase);
        } else {
          if (odd) build_cols<kHalfCols, kWords, KH, KW, CI, DW, true>(src, e0, tap_step, abase);
          else build_cols<kHalfCols, kWords, KH, KW, CI, DW, false>(src, e0, tap_step, abase);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[slot]);  // raw rows consumed (values are in TMEM / registers)
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[ab]);
        if (tr) trace[642 + 3 * pi] = clock64();
        ++pi;
        if (++slot == static_cast<uint32_t>(S)) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == kRpMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // Accumulators live in a ring of nacc BN-column slots, one per output depth
    // in flight (output depth g of the CTA's sequence -> slot g % nacc): a
    // plane feeds up to ceil(KD/sd) depths, and the slot of a finished depth is
    // drained by the epilogue while the MMAs carry on with the next planes.
    const uint64_t b0 = smem_desc(smem_u32(sB), b_rows * Cfg::kBRowBytes, 8 * Cfg::kBRowBytes, Cfg::kBLayout);
    constexpr uint32_t kBk16 = (16 * Cfg::kBRowBytes) >> 4;  // one K16 step of B (descriptor units)
    if (static_cast<int>(blockIdx.x) < p.total_units) {
      mbar_wait(bfull, 0);
      tc_fence_after();
    }
    // the CTA's planes in order (the producers and builders walk the same sequence)
    int per_unit = 0;
    for (int di = plane_lo; di <= plane_hi; ++di) {
      int o0, o1;
      od_range(di, o0, o1);
      per_unit += o0 <= o1;
    }
    const int my_units = static_cast<int>(blockIdx.x) < p.total_units
                             ? (p.total_units - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                             : 0;
    const uint32_t nplanes = static_cast<uint32_t>(my_units * per_unit);
    bool first_unit = true;
    {
      for (uint32_t pi = 0; pi < nplanes; ++pi) {
        const uint32_t ab = pi % nabuf, use = pi / nabuf;
        // The tensor pipe takes the next MMA only about when the previous one starts,
        // so anything the issuing thread does between MMAs is a pipe bubble (measured:
        // ~100 cycles per depth and ~450 per plane of bookkeeping halved the MMA rate).
        // Everything of the plane — each depth's accumulator slot, B offset, first /
        // last flags, the slot waits — is settled before the first MMA; the issue is
        // then straight-line MMAs and commits.
        mbar_wait(&afull[ab], use & 1);
        tc_fence_after();
        if (trace && lane == 0 && pi < 128) trace[256 + 2 * pi] = clock64();
        if (first_unit && lane == 0) {
          trace_event(p.trace, TR_FIRST_FULL);
          first_unit = false;
        }
        // the plane's depths, B offsets, accumulator slots and first / last flags were
        // computed by its producer: straight-line MMAs from here (the tensor pipe takes
        // the next MMA only about when the previous one starts, so bookkeeping between
        // MMAs is a bubble: ~800 cycles per plane when the MMA thread did it itself)
        uint32_t w[12];
        if constexpr (D3) {
          const uint4* dsc = pdesc + (pi % kRpDescRing) * 3;
          const uint4 q0 = dsc[0], q1 = dsc[1], q2 = dsc[2];
          w[0] = q0.x, w[1] = q0.y, w[2] = q0.z, w[3] = q0.w, w[4] = q1.x, w[5] = q1.y;
          w[6] = q1.z, w[7] = q1.w, w[8] = q2.x, w[9] = q2.y, w[10] = q2.z, w[11] = q2.w;
        } else {  // one plane per tile: depth 0, kd 0, the tile's own ring slot
          w[0] = 1;
          w[1] = 0;
          w[2] = (pi % nacc) | (1u << 4) | (1u << 5) | (((pi / nacc) & 1u) << 6);
        }
        const int nod = static_cast<int>(w[0]);
        const uint32_t a = tmem_base + a_col + ab * kWords;
        if (elect_one()) {
          constexpr int kMaxOd = kRpMaxSlots - 1;
#pragma unroll
          for (int i = 0; i < kMaxOd; ++i) {
            if (i < nod) {
              const uint32_t fl = w[2 + 2 * i], sl = fl & 15u;
              const bool fst = (fl >> 4) & 1u, lst = (fl >> 5) & 1u;
              if (fst) {
                mbar_wait(&tempty[sl], ((fl >> 6) & 1u) ^ 1u);  // the slot's previous depth was drained
                tc_fence_after();
              }
              const uint32_t d = tmem_base + sl * BN;
              const uint64_t bk = b0 + w[1 + 2 * i];
#pragma unroll
              for (int st = 0; st < kSteps; ++st)
                umma_f16_ts(d, a + 8 * st, bk + st * kBk16, Cfg::kIdesc, (fst && st == 0) ? 0u : 1u);
              if (lst) umma_commit(&tfull[sl]);
            }
          }
          umma_commit(&afree[ab]);
        }
        __syncwarp();
        if (trace && lane == 0 && pi < 128) trace[257 + 2 * pi] = clock64();
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ epilogue (TMA store)
    // thread = TMEM lane = output pixel m of the tile: for each output depth in
    // order, tcgen05.ld 32 columns -> the pixel's line of a dense [R][Wt][32]
    // staging box (swizzled 16-byte chunks) -> one bulk tensor store per 32-column
    // chunk; double-buffered staging.
    pdl_wait();  // Y (and the bias) may still be used / produced by the preceding kernel
    const uint32_t q = warp;
    const int m = static_cast<int>(q * 32 + lane);
    const bool mine = m < p.R * p.Wt;
    const int line_bytes = p.out_f16 ? 64 : 128;
    // fused epilogue: lane j keeps bias[c0 + j] of each 32-column chunk (broadcast by shuffles)
    float bias_lane[BN / 32];
#pragma unroll
    for (int i = 0; i < BN / 32; ++i) bias_lane[i] = p.bias ? __ldg(p.bias + 32 * i + lane) : 0.0f;
    const bool epi_on = p.bias || p.act;
    uint32_t chunk = 0, ui = 0;
    int ubase = 0;
    bool first = true;
    for (int u = blockIdx.x; u < p.total_units; u += gridDim.x, ubase += p.od) {
      int n, th, tw;
      decompose(u, n, th, tw);
      for (int od = 0; od < p.od; ++od) {
        const int g = ubase + od;
        const uint32_t sl = static_cast<uint32_t>(g % nacc), sph = static_cast<uint32_t>(g / nacc) & 1u;
        mbar_wait_backoff(&tfull[sl], sph, p.backoff_ns);
        tc_fence_after();
        if (trace && threadIdx.x == 0 && ui < 64) trace[512 + 2 * ui] = clock64();
        if (first && threadIdx.x == 0) trace_event(p.trace, TR_FIRST_TFULL);
        first = false;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32, ++chunk) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((q * 32u) << 16) + sl * BN + c0, r);
          tmem_ld_wait();
          if (epi_on) {
            float* v = reinterpret_cast<float*>(r);
            if (p.bias) {
              const float bl = bias_lane[c0 / 32];
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] += __shfl_sync(0xffffffffu, bl, i);
            }
            epi_act_n<32>(v, p.act);
          }
          uint8_t* buf = epi + (chunk & 1) * p.stage_bytes;
          named_bar_sync(1, 128);  // buffer (chunk & 1) no longer read by an older store
          if (mine) {
            uint8_t* dst = buf + m * line_bytes;
            if (p.out_f16) {
#pragma unroll
              for (int cc = 0; cc < 4; ++cc) {
                uint4 o;
                __half2 h0 = __floats2half2_rn(__uint_as_float(r[8 * cc]), __uint_as_float(r[8 * cc + 1]));
                __half2 h1 = __floats2half2_rn(__uint_as_float(r[8 * cc + 2]), __uint_as_float(r[8 * cc + 3]));
                __half2 h2 = __floats2half2_rn(__uint_as_float(r[8 * cc + 4]), __uint_as_float(r[8 * cc + 5]));
                __half2 h3 = __floats2half2_rn(__uint_as_float(r[8 * cc + 6]), __uint_as_float(r[8 * cc + 7]));
                o.x = *reinterpret_cast<uint32_t*>(&h0);
                o.y = *reinterpret_cast<uint32_t*>(&h1);
                o.z = *reinterpret_cast<uint32_t*>(&h2);
                o.w = *reinterpret_cast<uint32_t*>(&h3);
                *reinterpret_cast<uint4*>(dst + ((cc ^ ((m >> 1) & 3)) << 4)) = o;  // SW64
              }
            } else {
#pragma unroll
              for (int cc = 0; cc < 8; ++cc)
                *reinterpret_cast<uint4*>(dst + ((cc ^ (m & 7)) << 4)) =
                    make_uint4(r[4 * cc], r[4 * cc + 1], r[4 * cc + 2], r[4 * cc + 3]);  // SW128
            }
          }
          fence_proxy_async_smem();
          named_bar_sync(2, 128);
          if (threadIdx.x == 0 && !(p.debug & 2)) {
            const int zo = n * p.od + od;
            if (p.store_mode == 2)
              tma_reduce_add_4d(&p.tmY, buf, c0, tw * p.Wt, th * p.R, zo);
            else
              tma_store_4d(&p.tmY, buf, c0, tw * p.Wt, th * p.R, zo);
            tma_store_commit();
            tma_store_wait_read<1>();
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[sl]);
        if (trace && threadIdx.x == 0 && ui < 64) trace[513 + 2 * ui] = clock64();
        ++ui;
      }
    }
    if (threadIdx.x == 0) {
      tma_store_wait_read<0>();  // smem reads done; the grid end flushes the writes
      if (p.trace) {
        tma_store_wait_all<0>();  // (trace only) the stores themselves complete
        trace_event(p.trace, TR_STORES_DONE);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kRpMmaWarp) tmem_dealloc(tmem_base, 512);
  if (threadIdx.x == 0) trace_event(p.trace, TR_EXIT);
}

// Packed weight panel: Bp[kd][kh * 2 * WPK + kw * CI + ci][co] = W[kd][kh][kw][ci][co], zero elsewhere
// (the layout of the TMEM K vector; Kp = 16 * ksteps rows per kd).
__global__ void pack_rowpack_weights_kernel(const uint16_t* __restrict__ w, uint16_t* __restrict__ y, int32_t kd,
                                            int32_t kh, int32_t kw, int32_t ci, int32_t co, int32_t wpk,
                                            int32_t kp) {
  const int64_t total = static_cast<int64_t>(kd) * kp * co;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t col = static_cast<int32_t>(i % co);
    const int64_t row = i / co;
    const int32_t d = static_cast<int32_t>(row / kp);
    const int32_t k = static_cast<int32_t>(row - static_cast<int64_t>(d) * kp);
    const int32_t t = k / (2 * wpk), e = k - t * 2 * wpk;
    uint16_t v = 0;
    if (t < kh && e < kw * ci) v = w[((static_cast<int64_t>(d) * kh + t) * kw * ci + e) * co + col];
    y[i] = v;
  }
}

}  // namespace tb
