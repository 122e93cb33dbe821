// igemm.cuh — the tensorized contraction kernel: one persistent, warp-specialised
// tcgen05 implicit-GEMM used for GMM, C1D, C2D, C3D, DIL, GRP and T2D.
//
// It replaces the reference's tensorized-block HostKernel body
// (/root/reference/proj/include/tir/interp.h:120, dispatched from
// src/interp.cc:360-383) for whole-op blocks, computing
//     Y[m, g*COg + n] (+)= sum_k A[m, k] * B_g[k, n]
// where for GMM A/B are the operands and for convolutions A is the im2col view
// of X (never materialised: TMA im2col descriptors generate each 128-pixel x
// box_ch-channel slab on the fly) and B the HWIO weights viewed as [taps*CIg, CO]
// (a zero-copy reshape).
//
// Roles (256 threads, 1 CTA per SM pass, grid = min(tiles, SMs*occupancy)):
//   warp 0      TMA producer: A slab(s) + B tile per 64-deep K stage into a
//               multi-stage smem ring (full/empty mbarriers, expect_tx bytes)
//   warp 1      MMA issuer: 4 x tcgen05.mma.kind::f16 (M=128, N=BN, K=16) per
//               stage into a TMEM fp32 accumulator; tcgen05.commit frees the slot
//   warp 2      TMEM allocator (2 accumulators x BN columns, double-buffered)
//   warps 4-7   epilogue: tcgen05.ld -> (+Yin) -> fp32/fp16 vector stores; the
//               second accumulator lets tile i's epilogue overlap tile i+1's MMAs
//
// K enumeration (must match the reference reduction domain, workloads.h:106-108):
// k = tap * CIg + c with tap = (kd, kh, kw) row-major and c fastest, i.e. the
// weight row index. Stages hold 64 consecutive k; a stage is 64/box_ch "pieces",
// each one im2col TMA load of box_ch channels for one tap.
#pragma once

#include "ptx.cuh"

namespace tb {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 256;
constexpr int kMaxSub = 4;

enum AMode : int32_t { A_TILED = 2, A_IM2COL3 = 3, A_IM2COL4 = 4, A_IM2COL5 = 5 };

// One implicit-GEMM problem. A transposed convolution is s^2 (or s^3) of these
// (sub-pixel classes), a forward conv / GMM exactly one.
struct SubProb {
  int32_t m_count;            // GEMM rows (output pixels of this class)
  int32_t tiles_m;            // ceil(m_count / 128)
  int32_t tile_begin;         // first global tile id
  int32_t gx, gy, gz;         // m = ((n*gz + z)*gy + y)*gx + x
  int32_t a_lo[3], a_st[3];   // im2col base coordinate (x=w,y=h,z=d) = lo + idx*st
  int32_t taps[3];            // taps per dim (x, y, z)
  int32_t a_dil[3];           // im2col offset per tap step
  int32_t w_base[3], w_step[3];  // weight tap coordinate = base + t*step
  int32_t num_pieces;         // taps * cb_per_tap
  int32_t num_stages;         // ceil(num_pieces / pieces_per_stage)
  int32_t o_st[3], o_b[3];    // output coordinate = idx*st + b (x, y, z)
};

struct alignas(64) IgemmParams {
  CUtensorMap tmA[kMaxSub];
  CUtensorMap tmB;
  SubProb sub[kMaxSub];
  int32_t num_sub;
  int32_t total_tiles;
  int32_t tiles_n;     // N tiles per group
  int32_t groups;
  int32_t a_mode;      // AMode
  int32_t a_box_ch;    // channels per A piece: 64 / 32 / 16 / 8
  int32_t cig;         // K extent per tap (CI / G); GMM: K
  int32_t cb_per_tap;  // ceil(cig / a_box_ch)
  int32_t b_contig;    // 1: one B TMA per stage (rows contiguous); 0: one per piece
  int32_t k_rows;      // rows of B (OOB rows read as zero)
  int32_t w_kx, w_ky;  // weight tap linearisation: ((wz*w_ky + wy)*w_kx + wx)
  int32_t cog;         // valid output columns per group
  int32_t ldy;         // Y row pitch in elements (CO, or GMM N)
  int32_t out_dims[3]; // OW, OH, OD
  int32_t accumulate;
  int32_t out_f16;
  int32_t stages;      // smem ring depth
  void* Y;
  const float* Yin;
};

template <int BN>
struct IgemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;          // 16 KB
  static constexpr int kBBytes = kBK * BN * 2;           // 64 rows x BN
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
  static constexpr int kBChunk = BN < 64 ? BN : 64;        // columns per B TMA box
  static constexpr int kBRowBytes = kBChunk * 2;           // 128 / 64 / 32
  static constexpr uint32_t kBLayout = kBRowBytes == 128 ? 2u : kBRowBytes == 64 ? 4u : 6u;
  static constexpr uint32_t kIdesc = idesc_f16_f32(kBM, BN, /*A K-major*/ 0, /*B MN-major*/ 1);
  static size_t smem_bytes(int stages) {
    return 1024 /*align slack*/ + static_cast<size_t>(stages) * kStageBytes + 256 /*barriers*/;
  }
};

__device__ __forceinline__ void decompose_tile(const IgemmParams& p, int tile, int& s, int& mt,
                                               int& g, int& nt) {
  s = 0;
#pragma unroll 1
  for (int i = 1; i < p.num_sub; ++i)
    if (tile >= p.sub[i].tile_begin) s = i;
  int local = tile - p.sub[s].tile_begin;
  nt = local % p.tiles_n;
  int rest = local / p.tiles_n;
  g = rest % p.groups;
  mt = rest / p.groups;
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    igemm_tc_kernel(const __grid_constant__ IgemmParams p) {
  using Cfg = IgemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(S) * Cfg::kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < p.num_sub; ++i) prefetch_tmap(&p.tmA[i]);
    prefetch_tmap(&p.tmB);
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, Cfg::kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int pieces_per_stage = kBK / p.a_box_ch;
  const uint32_t piece_bytes = kBM * p.a_box_ch * 2;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x) {
        int s, mt, g, nt;
        decompose_tile(p, tile, s, mt, g, nt);
        const SubProb& sp = p.sub[s];
        const CUtensorMap* tmA = &p.tmA[s];
        const int m0 = mt * kBM;
        int x = m0 % sp.gx, rest = m0 / sp.gx;
        int y = rest % sp.gy;
        rest /= sp.gy;
        int z = rest % sp.gz;
        int n = rest / sp.gz;
        const int cx = sp.a_lo[0] + x * sp.a_st[0];
        const int cy = sp.a_lo[1] + y * sp.a_st[1];
        const int cz = sp.a_lo[2] + z * sp.a_st[2];
        const int col0 = g * p.cog + nt * BN;
        const int tx_n = sp.taps[0], txy_n = sp.taps[0] * sp.taps[1];
        for (int st = 0; st < sp.num_stages; ++st, ++it) {
          const uint32_t slot = it % S, phase = (it / S) & 1;
          mbar_wait(&empty[slot], phase ^ 1);
          uint8_t* sA = smem + static_cast<size_t>(slot) * Cfg::kStageBytes;
          uint8_t* sB = sA + Cfg::kABytes;
          mbar_arrive_expect_tx(&full[slot], Cfg::kStageBytes);
          for (int j = 0; j < pieces_per_stage; ++j) {
            int pc = st * pieces_per_stage + j;
            const bool real = pc < sp.num_pieces;
            if (!real) pc = sp.num_pieces - 1;  // finite data; its B rows are zero
            const int tap = pc / p.cb_per_tap, cb = pc - tap * p.cb_per_tap;
            const int tx = tap % tx_n, ty = (tap / tx_n) % sp.taps[1], tz = tap / txy_n;
            const int c = g * p.cig + cb * p.a_box_ch;
            void* dA = sA + j * piece_bytes;
            if (p.a_mode == A_TILED) {
              tma_load_2d(dA, tmA, &full[slot], c, m0);
            } else if (p.a_mode == A_IM2COL4) {
              tma_im2col_4d(dA, tmA, &full[slot], c, cx, cy, n,
                            static_cast<uint16_t>(tx * sp.a_dil[0]),
                            static_cast<uint16_t>(ty * sp.a_dil[1]));
            } else if (p.a_mode == A_IM2COL3) {
              tma_im2col_3d(dA, tmA, &full[slot], c, cx, n, static_cast<uint16_t>(tx * sp.a_dil[0]));
            } else {
              tma_im2col_5d(dA, tmA, &full[slot], c, cx, cy, cz, n,
                            static_cast<uint16_t>(tx * sp.a_dil[0]),
                            static_cast<uint16_t>(ty * sp.a_dil[1]),
                            static_cast<uint16_t>(tz * sp.a_dil[2]));
            }
            if (!p.b_contig) {
              int row = p.k_rows;  // fully out of bounds -> zeros
              if (real) {
                const int wx = sp.w_base[0] + tx * sp.w_step[0];
                const int wy = sp.w_base[1] + ty * sp.w_step[1];
                const int wz = sp.w_base[2] + tz * sp.w_step[2];
                row = ((wz * p.w_ky + wy) * p.w_kx + wx) * p.cig + cb * p.a_box_ch;
              }
#pragma unroll
              for (int ch = 0; ch < BN / Cfg::kBChunk; ++ch)
                tma_load_2d(sB + ch * (kBK * Cfg::kBRowBytes) + j * p.a_box_ch * Cfg::kBRowBytes,
                            &p.tmB, &full[slot], col0 + ch * Cfg::kBChunk, row);
            }
          }
          if (p.b_contig) {
#pragma unroll
            for (int ch = 0; ch < BN / Cfg::kBChunk; ++ch)
              tma_load_2d(sB + ch * (kBK * Cfg::kBRowBytes), &p.tmB, &full[slot],
                          col0 + ch * Cfg::kBChunk, st * kBK);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t it = 0, local = 0;
      // A descriptor geometry per piece width.
      uint32_t a_layout, a_sbo, a_lbo;
      switch (p.a_box_ch) {
        case 64: a_layout = 2; a_sbo = 1024; a_lbo = 16; break;
        case 32: a_layout = 4; a_sbo = 512; a_lbo = 16; break;
        case 16: a_layout = 6; a_sbo = 256; a_lbo = 16; break;
        default: a_layout = 0; a_sbo = 128; a_lbo = 2048; break;  // 8 channels, paired pieces
      }
      for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x, ++local) {
        int s, mt, g, nt;
        decompose_tile(p, tile, s, mt, g, nt);
        const int nst = p.sub[s].num_stages;
        const uint32_t acc = local & 1, acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int st = 0; st < nst; ++st, ++it) {
          const uint32_t slot = it % S, phase = (it / S) & 1;
          mbar_wait(&full[slot], phase);
          tc_fence_after();
          const uint32_t aBase = smem_u32(smem + static_cast<size_t>(slot) * Cfg::kStageBytes);
          const uint32_t bBase = aBase + Cfg::kABytes;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            uint32_t aaddr;
            switch (p.a_box_ch) {
              case 64: aaddr = aBase + 32 * k; break;
              case 32: aaddr = aBase + (k >> 1) * 8192 + (k & 1) * 32; break;
              case 16: aaddr = aBase + k * 4096; break;
              default: aaddr = aBase + k * 4096; break;  // pieces 2k, 2k+1 (2 KB each)
            }
            const uint64_t adesc = smem_desc(aaddr, a_lbo, a_sbo, a_layout);
            const uint64_t bdesc = smem_desc(bBase + k * 16 * Cfg::kBRowBytes,
                                             /*LBO: next 64-col chunk*/ kBK * Cfg::kBRowBytes,
                                             /*SBO: next 8 K rows*/ 8 * Cfg::kBRowBytes,
                                             Cfg::kBLayout);
            umma_f16(tmem_d, adesc, bdesc, Cfg::kIdesc, (st | k) != 0);
          }
          umma_commit(&empty[slot]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;
    const uint32_t row = q * 32 + lane;
    uint32_t local = 0;
    for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x, ++local) {
      int s, mt, g, nt;
      decompose_tile(p, tile, s, mt, g, nt);
      const SubProb& sp = p.sub[s];
      const uint32_t acc = local & 1, acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();

      const int m = mt * kBM + static_cast<int>(row);
      const bool row_ok = m < sp.m_count;
      int64_t pix = 0;
      if (row_ok) {
        int x = m % sp.gx, rest = m / sp.gx;
        int y = rest % sp.gy;
        rest /= sp.gy;
        int z = rest % sp.gz;
        int n = rest / sp.gz;
        const int ox = x * sp.o_st[0] + sp.o_b[0];
        const int oy = y * sp.o_st[1] + sp.o_b[1];
        const int oz = z * sp.o_st[2] + sp.o_b[2];
        pix = ((static_cast<int64_t>(n) * p.out_dims[2] + oz) * p.out_dims[1] + oy) *
                  p.out_dims[0] + ox;
      }
      const int ncol0 = nt * BN;  // within group
      const int64_t base = pix * p.ldy + g * p.cog + ncol0;
      constexpr int kChunk = BN < 32 ? BN : 32;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += kChunk) {
        uint32_t r[32];
        const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * BN + c0;
        if (kChunk == 32) tmem_ld_32x32b_x32(taddr, r);
        else tmem_ld_32x32b_x16(taddr, r);
        tmem_ld_wait();
        if (!row_ok) continue;
        const int valid = min(kChunk, p.cog - (ncol0 + c0));
        if (valid <= 0) continue;
        const int64_t off = base + c0;
        float v[32];
#pragma unroll
        for (int i = 0; i < kChunk; ++i) v[i] = __uint_as_float(r[i]);
        if (p.accumulate) {
          const float* yin = p.Yin + off;
          if (valid == kChunk && (off & 3) == 0) {
#pragma unroll
            for (int i = 0; i < kChunk; i += 4) {
              float4 t = *reinterpret_cast<const float4*>(yin + i);
              v[i] = t.x + v[i];
              v[i + 1] = t.y + v[i + 1];
              v[i + 2] = t.z + v[i + 2];
              v[i + 3] = t.w + v[i + 3];
            }
          } else {
            for (int i = 0; i < valid; ++i) v[i] = yin[i] + v[i];
          }
        }
        if (p.out_f16) {
          __half* y = reinterpret_cast<__half*>(p.Y) + off;
          if (valid == kChunk && (off & 7) == 0) {
#pragma unroll
            for (int i = 0; i < kChunk; i += 8) {
              uint4 u;
              __half2 h0 = __floats2half2_rn(v[i], v[i + 1]);
              __half2 h1 = __floats2half2_rn(v[i + 2], v[i + 3]);
              __half2 h2 = __floats2half2_rn(v[i + 4], v[i + 5]);
              __half2 h3 = __floats2half2_rn(v[i + 6], v[i + 7]);
              u.x = *reinterpret_cast<uint32_t*>(&h0);
              u.y = *reinterpret_cast<uint32_t*>(&h1);
              u.z = *reinterpret_cast<uint32_t*>(&h2);
              u.w = *reinterpret_cast<uint32_t*>(&h3);
              *reinterpret_cast<uint4*>(y + i) = u;
            }
          } else {
            for (int i = 0; i < valid; ++i) y[i] = __float2half_rn(v[i]);
          }
        } else {
          float* y = reinterpret_cast<float*>(p.Y) + off;
          if (valid == kChunk && (off & 3) == 0) {
#pragma unroll
            for (int i = 0; i < kChunk; i += 4)
              *reinterpret_cast<float4*>(y + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          } else {
            for (int i = 0; i < valid; ++i) y[i] = v[i];
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, Cfg::kTmemCols);
}

}  // namespace tb
