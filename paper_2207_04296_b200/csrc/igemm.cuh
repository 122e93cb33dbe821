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

// How B (weights) reaches shared memory:
//   B_STREAM    one TMA per K stage (rows of a stage are contiguous in B);
//   B_PIECES    one TMA per A piece (T2D: flipped taps are not contiguous);
//   B_RESIDENT  the whole [K, BN] panel is loaded once per CTA and stays in
//               smem (all tiles of a CTA share one (group, n-tile); host-checked).
enum BMode : int32_t { B_STREAM = 0, B_PIECES = 1, B_RESIDENT = 2 };

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
  int32_t b_mode;      // B_STREAM / B_PIECES / B_RESIDENT
  int32_t k_rows;      // rows of B (OOB rows read as zero)
  int32_t w_kx, w_ky;  // weight tap linearisation: ((wz*w_ky + wy)*w_kx + wx)
  int32_t cog;         // valid output columns per group
  int32_t ldy;         // Y row pitch in elements (CO, or GMM N)
  int32_t out_dims[3]; // OW, OH, OD
  int32_t accumulate;
  int32_t out_f16;
  int32_t stages;      // smem ring depth
  int32_t b_res_rows;  // B_RESIDENT: rows of the resident panel (multiple of 64)
  void* Y;
  const float* Yin;
  unsigned long long* trace;  // debug: per-stage clock64 stamps of CTA 0 (null in production)
};

template <int BN>
struct IgemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;          // 16 KB
  static constexpr int kBBytes = kBK * BN * 2;           // 64 rows x BN
  static constexpr int kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
  static constexpr int kBChunk = BN < 64 ? BN : 64;        // columns per B TMA box
  static constexpr int kBRowBytes = kBChunk * 2;           // 128 / 64 / 32
  static constexpr uint32_t kBLayout = kBRowBytes == 128 ? 2u : kBRowBytes == 64 ? 4u : 6u;
  static constexpr uint32_t kIdesc = idesc_f16_f32(kBM, BN, /*A K-major*/ 0, /*B MN-major*/ 1);
  // smem: [A ring: S x 16 KB][B ring: S x kBBytes | resident panel][barriers]
  static size_t smem_bytes(int stages, int b_res_rows) {
    const size_t b = b_res_rows ? static_cast<size_t>(b_res_rows) * BN * 2
                                : static_cast<size_t>(stages) * kBBytes;
    return 1024 /*align slack*/ + static_cast<size_t>(stages) * kABytes + b + 256 /*barriers*/;
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
  const bool b_res = p.b_mode == B_RESIDENT;
  uint8_t* sA0 = smem;
  uint8_t* sB0 = smem + static_cast<size_t>(S) * Cfg::kABytes;
  const size_t b_bytes = b_res ? static_cast<size_t>(p.b_res_rows) * BN * 2
                               : static_cast<size_t>(S) * Cfg::kBBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB0 + b_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint64_t* bres_full = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres_full + 1);

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
    mbar_init(bres_full, 1);
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

  unsigned long long* trace = (blockIdx.x == 0) ? p.trace : nullptr;
  if (trace && threadIdx.x == 0) trace[1023] = clock64();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // The whole warp runs the (warp-uniform) loop so addresses and coordinates
    // stay in uniform registers; one elected lane issues mbarrier/TMA ops.
    {
      const int box = p.a_box_ch;
      const int pps = kBK / box;
      const uint32_t piece_bytes = kBM * box * 2;
      const int cpt = p.cb_per_tap;
      const int a_mode = p.a_mode;
      const int b_mode = p.b_mode;
      const uint32_t stage_tx = Cfg::kABytes + (b_mode == B_RESIDENT ? 0u : Cfg::kBBytes);
      if (b_mode == B_RESIDENT && static_cast<int>(blockIdx.x) < p.total_tiles && elect_one()) {
        // Whole [b_res_rows, BN] panel of this CTA's (group, n-tile), once.
        int s0, mt0, g0, nt0;
        decompose_tile(p, blockIdx.x, s0, mt0, g0, nt0);
        const int col0 = g0 * p.cog + nt0 * BN;
        mbar_arrive_expect_tx(bres_full, static_cast<uint32_t>(p.b_res_rows) * BN * 2);
        for (int r = 0; r < p.b_res_rows; r += kBK)
#pragma unroll
          for (int ch = 0; ch < BN / Cfg::kBChunk; ++ch)
            tma_load_2d(sB0 + static_cast<size_t>(ch) * p.b_res_rows * Cfg::kBRowBytes +
                            static_cast<size_t>(r) * Cfg::kBRowBytes,
                        &p.tmB, bres_full, col0 + ch * Cfg::kBChunk, r);
      }
      uint32_t slot = 0, phase = 0;
      int it = 0;
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
        const int n = rest / sp.gz;
        const int cx = sp.a_lo[0] + x * sp.a_st[0];
        const int cy = sp.a_lo[1] + y * sp.a_st[1];
        const int cz = sp.a_lo[2] + z * sp.a_st[2];
        const int col0 = g * p.cog + nt * BN;
        const int T0 = sp.taps[0], T1 = sp.taps[1];
        const int dx = sp.a_dil[0], dy = sp.a_dil[1], dz = sp.a_dil[2];
        const int npieces = sp.num_pieces, nst = sp.num_stages;
        const int cbase = g * p.cig;
        // piece state: channel block, tap (tx, ty, tz), im2col offsets
        int cb = 0, tx = 0, ty = 0, tz = 0, ox = 0, oy = 0, oz = 0, pc = 0;
        for (int st = 0; st < nst; ++st, ++it) {
          mbar_wait(&empty[slot], phase ^ 1);
          if (trace && lane == 0 && it < 128) trace[2 * it] = clock64();
          uint8_t* sA = sA0 + slot * Cfg::kABytes;
          uint8_t* sB = sB0 + slot * Cfg::kBBytes;
          const bool leader = elect_one();
          if (leader) mbar_arrive_expect_tx(&full[slot], stage_tx);
          if (trace && lane == 0 && it < 64) trace[768 + 4 * it] = clock64();
          for (int j = 0; j < pps; ++j) {
            const int c = cbase + cb * box;
            void* dA = sA + j * piece_bytes;
            if (!leader) {
            } else if (a_mode == A_IM2COL4) {
              tma_im2col_4d(dA, tmA, &full[slot], c, cx, cy, n, static_cast<uint16_t>(ox),
                            static_cast<uint16_t>(oy));
            } else if (a_mode == A_TILED) {
              tma_load_2d(dA, tmA, &full[slot], c, m0);
            } else if (a_mode == A_IM2COL3) {
              tma_im2col_3d(dA, tmA, &full[slot], c, cx, n, static_cast<uint16_t>(ox));
            } else {
              tma_im2col_5d(dA, tmA, &full[slot], c, cx, cy, cz, n, static_cast<uint16_t>(ox),
                            static_cast<uint16_t>(oy), static_cast<uint16_t>(oz));
            }
            if (trace && lane == 0 && it < 64 && j == 0) trace[768 + 4 * it + 1] = clock64();
            if (b_mode == B_PIECES) {
              int row = p.k_rows;  // beyond the last piece: fully out of bounds -> zeros
              if (pc < npieces) {
                const int wx = sp.w_base[0] + tx * sp.w_step[0];
                const int wy = sp.w_base[1] + ty * sp.w_step[1];
                const int wz = sp.w_base[2] + tz * sp.w_step[2];
                row = ((wz * p.w_ky + wy) * p.w_kx + wx) * p.cig + cb * box;
              }
              if (leader)
#pragma unroll
                for (int ch = 0; ch < BN / Cfg::kBChunk; ++ch)
                  tma_load_2d(sB + ch * (kBK * Cfg::kBRowBytes) + j * box * Cfg::kBRowBytes,
                              &p.tmB, &full[slot], col0 + ch * Cfg::kBChunk, row);
            }
            // Advance to the next piece; past the end, keep re-reading the last
            // real A piece (finite data) whose B rows are zero.
            ++pc;
            if (pc < npieces) {
              if (++cb == cpt) {
                cb = 0;
                ox += dx;
                if (++tx == T0) {
                  tx = 0;
                  ox = 0;
                  oy += dy;
                  if (++ty == T1) {
                    ty = 0;
                    oy = 0;
                    oz += dz;
                    ++tz;
                  }
                }
              }
            }
          }
          if (trace && lane == 0 && it < 64) trace[768 + 4 * it + 2] = clock64();
          if (b_mode == B_STREAM && leader) {
#pragma unroll
            for (int ch = 0; ch < BN / Cfg::kBChunk; ++ch)
              tma_load_2d(sB + ch * (kBK * Cfg::kBRowBytes), &p.tmB, &full[slot],
                          col0 + ch * Cfg::kBChunk, st * kBK);
          }
          if (trace && lane == 0 && it < 64) trace[768 + 4 * it + 3] = clock64();
          __syncwarp();
          if (trace && lane == 0 && it < 128) trace[2 * it + 1] = clock64();
          if (++slot == static_cast<uint32_t>(S)) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Warp-uniform loop; one elected lane issues tcgen05.mma / commit.
    {
      // Descriptor templates; per stage/k only the 14-bit start-address field
      // (bits 0-13, address >> 4) changes, so plain 64-bit adds update it.
      uint32_t a_layout, a_sbo, a_lbo;
      uint32_t a_koff[4];  // byte offset of k-step k within an A stage
      switch (p.a_box_ch) {
        case 64:
          a_layout = 2; a_sbo = 1024; a_lbo = 16;
          for (int k = 0; k < 4; ++k) a_koff[k] = 32 * k;
          break;
        case 32:
          a_layout = 4; a_sbo = 512; a_lbo = 16;
          for (int k = 0; k < 4; ++k) a_koff[k] = (k >> 1) * 8192 + (k & 1) * 32;
          break;
        case 16:
          a_layout = 6; a_sbo = 256; a_lbo = 16;
          for (int k = 0; k < 4; ++k) a_koff[k] = k * 4096;
          break;
        default:  // 8 channels: pieces 2k and 2k+1 form one K=16 step (no swizzle)
          a_layout = 0; a_sbo = 128; a_lbo = 2048;
          for (int k = 0; k < 4; ++k) a_koff[k] = k * 4096;
          break;
      }
      const uint64_t adesc0 = smem_desc(smem_u32(sA0), a_lbo, a_sbo, a_layout);
      const uint32_t b_lbo = b_res ? p.b_res_rows * Cfg::kBRowBytes : kBK * Cfg::kBRowBytes;
      const uint64_t bdesc0 = smem_desc(smem_u32(sB0), b_lbo, 8 * Cfg::kBRowBytes, Cfg::kBLayout);
      constexpr uint32_t kBk = (16 * Cfg::kBRowBytes) >> 4;   // per k-step (16 rows)
      constexpr uint32_t kBst = (kBK * Cfg::kBRowBytes) >> 4; // per 64-row stage (resident)
      constexpr uint32_t kBslot = Cfg::kBBytes >> 4;          // per ring slot (streamed)
      constexpr uint32_t kAslot = Cfg::kABytes >> 4;
      if (b_res && static_cast<int>(blockIdx.x) < p.total_tiles) {
        mbar_wait(bres_full, 0);
        tc_fence_after();
      }
      uint32_t slot = 0, phase = 0, local = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x, ++local) {
        int s, mt, g, nt;
        decompose_tile(p, tile, s, mt, g, nt);
        const int nst = p.sub[s].num_stages;
        const uint32_t acc = local & 1, acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int st = 0; st < nst; ++st, ++it) {
          mbar_wait(&full[slot], phase);
          tc_fence_after();
          if (trace && lane == 0 && it < 128) trace[256 + 2 * it] = clock64();
          const uint64_t a = adesc0 + slot * kAslot;
          const uint64_t b = bdesc0 + (b_res ? st * kBst : slot * kBslot);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_f16(tmem_d, a + (a_koff[k] >> 4), b + k * kBk, Cfg::kIdesc, (st | k) != 0);
            umma_commit(&empty[slot]);
          }
          __syncwarp();
          if (trace && lane == 0 && it < 128) trace[256 + 2 * it + 1] = clock64();
          if (++slot == static_cast<uint32_t>(S)) {
            slot = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit(&tfull[acc]);
        __syncwarp();
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
      if (trace && threadIdx.x == 128 && local < 64) trace[512 + 2 * local] = clock64();

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
        const int valid = min(kChunk, p.cog - (ncol0 + c0));
        if (!row_ok || valid <= 0) continue;
        const int64_t off = base + c0;
        float v[kChunk];
#pragma unroll
        for (int i = 0; i < kChunk; ++i) v[i] = __uint_as_float(r[i]);
        const bool full_vec = valid == kChunk && (off & 7) == 0;
        if (p.accumulate) {
          const float* yin = p.Yin + off;
          if (full_vec) {
#pragma unroll
            for (int i = 0; i < kChunk; i += 4) {
              const float4 t = *reinterpret_cast<const float4*>(yin + i);
              v[i] = t.x + v[i];
              v[i + 1] = t.y + v[i + 1];
              v[i + 2] = t.z + v[i + 2];
              v[i + 3] = t.w + v[i + 3];
            }
          } else {
#pragma unroll
            for (int i = 0; i < kChunk; ++i)
              if (i < valid) v[i] = yin[i] + v[i];
          }
        }
        if (p.out_f16) {
          __half* y = reinterpret_cast<__half*>(p.Y) + off;
          if (full_vec) {
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
#pragma unroll
            for (int i = 0; i < kChunk; ++i)
              if (i < valid) y[i] = __float2half_rn(v[i]);
          }
        } else {
          float* y = reinterpret_cast<float*>(p.Y) + off;
          if (full_vec) {
#pragma unroll
            for (int i = 0; i < kChunk; i += 4)
              *reinterpret_cast<float4*>(y + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < kChunk; ++i)
              if (i < valid) y[i] = v[i];
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (trace && threadIdx.x == 128 && local < 64) trace[512 + 2 * local + 1] = clock64();
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, Cfg::kTmemCols);
}

}  // namespace tb
