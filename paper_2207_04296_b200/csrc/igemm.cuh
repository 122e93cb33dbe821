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
// Stages hold KS sub-blocks of 64 K (KS = 1, 2 or 4, a template parameter):
// one barrier round then covers 4*KS MMAs, amortising the ~400-cycle
// wait/commit latency of the single MMA warp (tools/trace_igemm.py).
//
// Roles (288 threads = 9 warps, persistent, grid = min(tiles, SMs)):
//   warps 0-3   epilogue: tcgen05.ld -> (+Yin) -> fp32/fp16 vector stores; the
//               second accumulator lets tile i's epilogue overlap tile i+1's MMAs
//               (warp w reads TMEM lanes 32*(w%4)..+31)
//   warps 4-7   TMA producers: producer w fills stages st = w, w+4, ... of every
//               tile (A slab(s) + B tile per 64-deep K stage) into one shared
//               smem ring (full/empty mbarriers, expect_tx bytes). Measured on
//               B200 (tools/l2bw.cu): an issuing thread completes about one TMA
//               request per ~500 cycles regardless of its queue depth, while
//               independent issuers scale linearly to the ~17 TB/s L2 roof — so
//               the loads are spread over four issuers.
//   warp 8      TMEM allocator + MMA issuer: 4 x tcgen05.mma.kind::f16
//               (M=128, N=BN, K=16) per stage into a TMEM fp32 accumulator;
//               tcgen05.commit frees the slot / publishes the accumulator
// The EPI8 instantiation (384 threads: 8 epilogue + 3 producer + 1 MMA warps,
// IgemmCfg) splits each tile's columns over two epilogue warps per TMEM
// sub-partition; the host picks it for short-K fused tiles (use_epi8).
//
// K enumeration (must match the reference reduction domain, workloads.h:106-108):
// k = tap * CIg + c with tap = (kd, kh, kw) row-major and c fastest, i.e. the
// weight row index. Stages hold 64 consecutive k; a stage is 64/box_ch "pieces",
// each one im2col TMA load of box_ch channels for one tap.
#pragma once

#include "ptx.cuh"

namespace tb {

constexpr int kBM = 128;
constexpr int kBK = 64;  // K per sub-block (one 128-byte swizzle row of fp16)
constexpr int kThreads = 288;  // 4 epilogue + 4 producer + 1 MMA warps (EPI8: 8 + 3 + 1 = 384)
constexpr int kMaxPieces = 2048;  // per-launch piece table entries (16 B each)
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
  int32_t piece_begin;        // offset of this sub-problem in the piece table
  int32_t o_st[3], o_b[3];    // output coordinate = idx*st + b (x, y, z)
};

// Batched GMM (attention): problem z = z1 * z2n + z2 reads A_z[m, k] =
// A[ar(z) + m, ac(z) + k], B_z[k, n] = B[br(z) + k, bc(z) + n] and writes
// C_z[m, n] = C[cr(z) + m, cc(z) + n], each coordinate base + z1*step1 + z2*step2
// over plain 2-D tensor maps (strided heads / batches need no copies).
struct BatchAxis {
  int32_t row[3], col[3];  // base, per-z1 step, per-z2 step
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
  const float* bias;  // fused epilogue: per-output-column bias (nullable)
  int32_t relu;       // fused epilogue activation (1 ReLU, 2 ReLU6, 3 GELU)
  const uint16_t* residual;  // fused epilogue: fp16 residual in Y's layout
  int32_t out_f16;
  int32_t stages;      // smem ring depth
  int32_t b_res_rows;  // B_RESIDENT: rows of the resident panel (multiple of 64)
  int32_t total_pieces;  // piece-table entries (sum of sub-problem num_pieces)
  void* Y;
  const float* Yin;
  int32_t store_mode;  // 0: generic row-offset stores, 1: TMA store, 2: TMA reduce-add (Y += tile)
  int32_t epi_cw;      // store modes 1/2: columns per staged chunk (32, or 64 for fp16 with BN >= 64)
  int32_t bias_floats; // > 0: the whole bias vector is staged in shared memory (16-byte broadcasts)
  int32_t ksplit;      // split-K partitions (>= 1); > 1: clusters of ksplit CTAs, one output tile each,
                       // partials combined through distributed shared memory (see cluster_reduce)
  CUtensorMap tmY;     // store_mode != 0: Y as 2-D [rows, ldy], box {32, 32}
  unsigned long long* trace;  // debug: per-stage clock64 stamps of CTA 0 (null in production)
  int32_t batch_tiles;  // batched GMM: tiles per problem (0 = not batched)
  int32_t b_kmajor;     // B given as [N rows, K cols] (K contiguous): K-major UMMA operand, SW128
                        // boxes {64 K, BN rows} (attention's Q K^T reads K straight from QKV)
  int32_t mc;           // 2: cta_group::2 CTA pair (CG2 instantiation, clusters of 2): see mc_tile
  int32_t batch_z2;     // problems per z1
  int32_t l2_prefetch;  // producers prefetch their share of the first stage's A into L2 before the PDL wait
  int32_t gp_taps, gp_kpg;  // GP instantiation (group-packed): taps, K16 steps per packed group (cig / 16)
  BatchAxis ba, bb, bc; // A / B / C coordinates per problem
};

// Splits a batched tile id into (problem-local tile, z1, z2).
__device__ __forceinline__ void split_batch(const IgemmParams& p, int& tile, int& z1, int& z2) {
  z1 = z2 = 0;
  if (p.batch_tiles) {
    const int z = tile / p.batch_tiles;
    tile -= z * p.batch_tiles;
    z1 = z / p.batch_z2;
    z2 = z - z1 * p.batch_z2;
  }
}

__device__ __forceinline__ int batch_row(const BatchAxis& a, int z1, int z2) {
  return a.row[0] + z1 * a.row[1] + z2 * a.row[2];
}
__device__ __forceinline__ int batch_col(const BatchAxis& a, int z1, int z2) {
  return a.col[0] + z1 * a.col[1] + z2 * a.col[2];
}

// EPI8: the short-K variant (1x1 convs / expansion GEMMs / attention, whose
// tiles are a few MMAs and a 128 x BN epilogue): 8 epilogue warps — two per TMEM
// lane quadrant, alternating column chunks — so two epilogue warps share each
// SM sub-partition and overlap their latency-bound chunk chains; 3 producers
// suffice for one or two stages per tile.
// GP (group-packed): a 64-channel im2col piece carries 64 / cig groups of a grouped
// conv (cig = 16 or 32); the tile's BN columns are those groups' 32 output columns
// each, every MMA is N = 32 on its group's K16 steps, B is the [taps*cig, 32] panel
// of each group (32-column SW64 chunks). One TMA request per tap feeds all the
// packed groups instead of one narrow request per group.
template <int BN, int KS, bool EPI8 = false, bool GP = false>
struct IgemmCfg {
  static constexpr int kEpiWarps = EPI8 ? 8 : 4;
  static constexpr int kProd = EPI8 ? 3 : 4;
  static constexpr int kMma = kEpiWarps + kProd;          // MMA warp (last)
  static constexpr int kThreadsN = 32 * (kMma + 1);
  static constexpr int kSubA = kBM * kBK * 2;               // 16 KB per 64-deep sub-block
  static constexpr int kABytes = KS * kSubA;
  static constexpr int kBRows = KS * kBK;                   // B rows per stage
  static constexpr int kBBytes = kBRows * BN * 2;
  static constexpr int kNacc = (4 * BN <= 512) ? 4 : 2;     // TMEM accumulator buffers
  static constexpr int kTmemCols = (kNacc * BN <= 32) ? 32 : (kNacc * BN <= 64) ? 64
                                   : (kNacc * BN <= 128) ? 128 : (kNacc * BN <= 256) ? 256 : 512;
  static constexpr int kBChunk = GP ? 32 : BN < 64 ? BN : 64;  // columns per B TMA box
  static constexpr int kBRowBytes = kBChunk * 2;           // 128 / 64 / 32
  static constexpr uint32_t kBLayout = kBRowBytes == 128 ? 2u : kBRowBytes == 64 ? 4u : 6u;
  static constexpr uint32_t kIdesc = idesc_f16_f32(kBM, GP ? 32 : BN, /*A K-major*/ 0, /*B MN-major*/ 1);
  // epilogue staging: per epilogue warp two 4 KB buffers (32 rows x 32 fp32)
  static constexpr int kEpiWarpBytes = 8192;
  static constexpr int kEpiBytes = kEpiWarps * kEpiWarpBytes;
  // smem: [A ring][B ring | resident panel][epilogue staging][piece table][barriers]
  static size_t smem_bytes(int stages, int b_res_rows, int pieces, int bias_floats, bool cg2 = false) {
    const size_t b = b_res_rows ? static_cast<size_t>(b_res_rows) * BN * 2
                                : static_cast<size_t>(stages) * (cg2 ? kBBytes / 2 : kBBytes);
    return 1024 /*align slack*/ + static_cast<size_t>(stages) * kABytes + b + kEpiBytes +
           static_cast<size_t>(pieces) * sizeof(int4) + static_cast<size_t>(bias_floats) * 4 + 256 /*barriers*/;
  }
};

// tile -> (sub-problem, m tile, group, n tile, K split); the split index is
// fastest so a persistent CTA keeps one (group, n tile) when
// grid % (ksplit * groups * tiles_n) == 0 (resident-B requirement).
__device__ __forceinline__ void decompose_tile(const IgemmParams& p, int tile, int& s, int& mt,
                                               int& g, int& nt, int& ks) {
  s = 0;
#pragma unroll 1
  for (int i = 1; i < p.num_sub; ++i)
    if (tile >= p.sub[i].tile_begin) s = i;
  int local = tile - p.sub[s].tile_begin;
  ks = local % p.ksplit;
  local /= p.ksplit;
  nt = local % p.tiles_n;
  int rest = local / p.tiles_n;
  g = rest % p.groups;
  mt = rest / p.groups;
}

// CTA pairs (CG2; GMM-shaped launches only: one sub-problem, one group, no
// split-K or batch, even M-tile count). The grid is clusters of 2 and CTA r of a
// cluster takes M tile 2*i + r of the same N tile as its peer. Iteration tile t
// (t = blockIdx.x + j * gridDim.x, gridDim even) -> pair t / 2, rank t & 1.
template <bool CG2>
__device__ __forceinline__ int mc_tile(const IgemmParams& p, int tile) {
  if constexpr (!CG2) {
    return tile;
  } else {
    const int pt = tile >> 1;
    const int nt = pt % p.tiles_n, mtp = pt / p.tiles_n;
    return (2 * mtp + (tile & 1)) * p.tiles_n + nt;
  }
}

// The pair runs tcgen05.mma.cta_group::2 (M = 256, the leader issues
// for both CTAs). Each CTA loads its own A and HALF of B's columns (no
// multicast), so per-SM shared-memory fill and MMA operand reads both drop to
// A + B/2; TMA loads complete on the leader's full barrier, commits multicast.
__device__ __forceinline__ uint32_t mc_leader_addr(const void* q) { return smem_u32(q) & 0xFEFFFFFFu; }

__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* m, uint32_t leader_bar, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void umma_f16_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit_cg2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_rank0(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

__device__ __forceinline__ void mc_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void decompose_tile(const IgemmParams& p, int tile, int& s, int& mt,
                                               int& g, int& nt) {
  int ks;
  decompose_tile(p, tile, s, mt, g, nt, ks);
}

// Stage range [st0, st1) of split `ks` out of `nst` stages.
__device__ __forceinline__ void split_range(const IgemmParams& p, int nst, int ks, int& st0, int& st1) {
  st0 = static_cast<int>(static_cast<int64_t>(nst) * ks / p.ksplit);
  st1 = static_cast<int>(static_cast<int64_t>(nst) * (ks + 1) / p.ksplit);
}

__device__ __forceinline__ float4 ld_cluster_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// Output element offset of each row this cluster rank combines (-1: past the
// sub-problem), written to row_off[0, rows) by threads [0, nthr). The epilogue warps
// call it while the MMAs run, so the combine finds its row offsets ready.
template <int BN>
__device__ __forceinline__ void split_row_offsets(const IgemmParams& p, int64_t* row_off, int tid, int nthr) {
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tile = blockIdx.x;
  if (tile >= p.total_tiles) return;
  int s = 0, mt = 0, g = 0, nt = 0, kk = 0;
  decompose_tile(p, tile, s, mt, g, nt, kk);
  const SubProb& sp = p.sub[s];
  const int rows = (kBM + p.ksplit - 1) / p.ksplit;
  const int r0 = static_cast<int>(rank) * rows, r1 = min(kBM, r0 + rows);
  // the combine's tile coordinates, after the (at most 64) row offsets: decompose_tile's
  // dependent constant loads and divisions cost ~0.45 us when the combine starts
  if (tid == 0) {
    int* meta = reinterpret_cast<int*>(row_off + kBM / 2);
    meta[0] = g;
    meta[1] = nt;
    meta[2] = r0;
    meta[3] = r1;
  }
  for (int r = r0 + tid; r < r1; r += nthr) {
    const int m = mt * kBM + r;
    int64_t off = -1;
    if (m < sp.m_count) {
      int x = m % sp.gx, rest = m / sp.gx;
      const int y = rest % sp.gy;
      rest /= sp.gy;
      const int z = rest % sp.gz;
      const int n = rest / sp.gz;
      const int64_t pix = ((static_cast<int64_t>(n) * p.out_dims[2] + z * sp.o_st[2] + sp.o_b[2]) * p.out_dims[1] +
                           y * sp.o_st[1] + sp.o_b[1]) * p.out_dims[0] + x * sp.o_st[0] + sp.o_b[0];
      off = pix * p.ldy + g * p.cog + nt * BN;
    }
    row_off[r - r0] = off;
  }
}

// One rank's share of the split-K combine: passes of KU items (float4 of the
// partial rows [r0, r1)) per thread, every split's load of a pass in flight at
// once; the cluster barrier is ARRIVED as soon as the last pass's remote loads
// have been consumed (peers may then exit), and WAITED after the stores.
template <int BN, int KMAX, int KU>
__device__ __forceinline__ void cluster_combine(const IgemmParams& p, uint32_t base, const int64_t* row_off, int r0,
                                                int r1, int g, int nt, bool active) {
  constexpr int kV = BN / 4;  // float4 per partial row
  const int ks = p.ksplit;
  const int valid = p.cog - nt * BN;
  const bool vec_ok = (p.ldy % 8 == 0) && (p.cog % 8 == 0) && ((reinterpret_cast<uintptr_t>(p.Y) & 15) == 0) &&
                      (!p.accumulate || (reinterpret_cast<uintptr_t>(p.Yin) & 15) == 0);
  const int items = active ? (r1 - r0) * kV : 0;
  const int per_pass = KU * static_cast<int>(blockDim.x);
  const int passes = (items + per_pass - 1) / per_pass;  // CTA-uniform
  if (passes == 0) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  if (active) pdl_wait();  // Yin / residual may come from the preceding kernel
  if (threadIdx.x == 0) trace_x(p.trace, 6);
#pragma unroll 1
  for (int pass = 0; pass < passes; ++pass) {
    const int i0 = pass * per_pass + static_cast<int>(threadIdx.x);
    float4 t[KMAX][KU];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k < ks) {
        uint32_t rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(base), "r"(k));
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          const int i = i0 + u * static_cast<int>(blockDim.x);
          if (i < items) {
            const int row = r0 + i / kV, col = (i % kV) * 4;
            t[k][u] = ld_cluster_f4(rb + static_cast<uint32_t>((row * (BN + 4) + col) * 4));
          }
        }
      }
    }
    float4 v[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      v[u] = t[0][u];
#pragma unroll
      for (int k = 1; k < KMAX; ++k) {  // fixed order ((p_0 + p_1) + p_2) + ...
        if (k < ks) {
          v[u].x = v[u].x + t[k][u].x; v[u].y = v[u].y + t[k][u].y;
          v[u].z = v[u].z + t[k][u].z; v[u].w = v[u].w + t[k][u].w;
        }
      }
    }
    if (pass == passes - 1) {  // every remote read of this CTA is done (the sums consumed them)
      if (threadIdx.x == 0) trace_x(p.trace, 7);
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int i = i0 + u * static_cast<int>(blockDim.x);
      if (i >= items) continue;
      const int row = i / kV, col = (i % kV) * 4;
      const int64_t ro = row_off[row];
      if (ro < 0 || col >= valid) continue;
      const int64_t off = ro + col;
      const int lim = valid - col;
      const bool vec = vec_ok && lim >= 4;
      float* vv = reinterpret_cast<float*>(&v[u]);
      if (p.accumulate) {
        if (vec) {
          const float4 y0 = *reinterpret_cast<const float4*>(p.Yin + off);
          vv[0] = y0.x + vv[0]; vv[1] = y0.y + vv[1]; vv[2] = y0.z + vv[2]; vv[3] = y0.w + vv[3];
        } else {
          for (int j = 0; j < 4 && j < lim; ++j) vv[j] = p.Yin[off + j] + vv[j];
        }
      }
      if (p.bias || p.relu || p.residual)
        epi_run<4>(vv, p.bias, g * p.cog + nt * BN + col, lim, p.residual ? p.residual + off : nullptr, p.relu);
      if (p.out_f16) {
        __half* yp = reinterpret_cast<__half*>(p.Y) + off;
        if (vec) {
          __half2 h0 = __floats2half2_rn(vv[0], vv[1]), h1 = __floats2half2_rn(vv[2], vv[3]);
          uint2 w2;
          w2.x = *reinterpret_cast<uint32_t*>(&h0);
          w2.y = *reinterpret_cast<uint32_t*>(&h1);
          *reinterpret_cast<uint2*>(yp) = w2;
        } else {
          for (int j = 0; j < 4 && j < lim; ++j) yp[j] = __float2half_rn(vv[j]);
        }
      } else {
        float* yp = reinterpret_cast<float*>(p.Y) + off;
        if (vec) *reinterpret_cast<float4*>(yp) = v[u];
        else
          for (int j = 0; j < 4 && j < lim; ++j) yp[j] = vv[j];
      }
    }
  }
}

// Deterministic split-K. The ksplit CTAs of a cluster (consecutive tile ids:
// the split index is fastest) hold the fp32 partials of ONE output tile in
// shared memory ([128][BN + 4], written by the epilogue warps). After a cluster
// barrier, cluster rank r combines rows [r*R, (r+1)*R) of the tile over all
// ranks through distributed shared memory in the fixed order
// ((p_0 + p_1) + p_2) + ..., then applies the C-ABI epilogue — (Yin +) sum,
// + bias, + residual, activation — and stores 16-byte vectors at the output
// pixel of each row (row-linear or, for T2D classes, strided). No memset, no
// atomics: the result is identical on every run. A second barrier keeps every
// partial alive until all ranks have read it. All threads of the CTA take part.
template <int BN>
__device__ __forceinline__ void cluster_reduce(const IgemmParams& p, const float* part, int64_t* row_off) {
  if (threadIdx.x == 0) trace_x(p.trace, 0);
  mc_cluster_sync();  // every partial of the cluster is written (release / acquire)
  if (threadIdx.x == 0) trace_x(p.trace, 1);
  const int ks = p.ksplit;
  const bool active = static_cast<int>(blockIdx.x) < p.total_tiles;
  // row_off[] and the tile coordinates were written by the epilogue warps
  // (split_row_offsets) before the kernel-end barrier
  const int* meta = reinterpret_cast<const int*>(row_off + kBM / 2);
  const int g = active ? meta[0] : 0, nt = active ? meta[1] : 0;
  const int r0 = active ? meta[2] : 0, r1 = active ? meta[3] : 0;
  if (threadIdx.x == 0) trace_x(p.trace, 2);
  const uint32_t base = smem_u32(part);
  if (ks <= 2) cluster_combine<BN, 2, 4>(p, base, row_off, r0, r1, g, nt, active);
  else if (ks <= 4) cluster_combine<BN, 4, 2>(p, base, row_off, r0, r1, g, nt, active);
  else cluster_combine<BN, 8, 2>(p, base, row_off, r0, r1, g, nt, active);
  if (threadIdx.x == 0) trace_event(p.trace, TR_STORES_DONE);
  // peers have finished reading this CTA's partial (arrived in cluster_combine)
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) trace_x(p.trace, 3);
}

// Piece table entry: everything a producer needs for one TMA piece, computed
// once per launch so the producer loop does no index arithmetic.
//   x = channel offset within the group (cb * box)
//   y = im2col offsets ox | oy << 16,   z = oz
//   w = B row (B_PIECES: weight row of this tap/channel block)
__device__ __forceinline__ int4 make_piece(const IgemmParams& p, const SubProb& sp, int pc) {
  const int cpt = p.cb_per_tap;
  const int tap = pc / cpt, cb = pc - tap * cpt;
  const int T0 = sp.taps[0], T1 = sp.taps[1];
  const int tx = tap % T0, ty = (tap / T0) % T1, tz = tap / (T0 * T1);
  const int wx = sp.w_base[0] + tx * sp.w_step[0];
  const int wy = sp.w_base[1] + ty * sp.w_step[1];
  const int wz = sp.w_base[2] + tz * sp.w_step[2];
  int4 e;
  e.x = cb * p.a_box_ch;
  e.y = (tx * sp.a_dil[0]) | ((ty * sp.a_dil[1]) << 16);
  e.z = tz * sp.a_dil[2];
  e.w = ((wz * p.w_ky + wy) * p.w_kx + wx) * p.cig + cb * p.a_box_ch;
  return e;
}

// CG2 instantiations (host p.mc == 2) contain cta_group::2 instructions and must be
// launched as clusters of 2; every other launch uses CG2 = false.
template <int BN, int KS, bool EPI8 = false, bool CG2 = false, bool GP = false>
__global__ void __launch_bounds__(IgemmCfg<BN, KS, EPI8>::kThreadsN, 1)
    igemm_tc_kernel(const __grid_constant__ IgemmParams p) {
  using Cfg = IgemmCfg<BN, KS, EPI8, GP>;
  constexpr int kProducers = Cfg::kProd;
  constexpr int kEpi = Cfg::kEpiWarps;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  if (threadIdx.x == 0) trace_event(p.trace, TR_ENTRY);
  const int S = p.stages;
  const bool b_res = p.b_mode == B_RESIDENT;
  constexpr int kBSlotBytes = CG2 ? Cfg::kBBytes / 2 : Cfg::kBBytes;  // cg2: this CTA's half of B
  uint8_t* sA0 = smem;
  uint8_t* sB0 = smem + static_cast<size_t>(S) * Cfg::kABytes;
  const size_t b_bytes = b_res ? static_cast<size_t>(p.b_res_rows) * BN * 2
                               : static_cast<size_t>(S) * kBSlotBytes;
  uint8_t* epi_smem = sB0 + b_bytes;  // 1024-aligned (all preceding sizes are)
  int4* pieces = reinterpret_cast<int4*>(epi_smem + Cfg::kEpiBytes);
  // staged fp32 bias (p.bias_floats columns; 0 = read from global with shuffles)
  float* sbias = reinterpret_cast<float*>(pieces + p.total_pieces);
  uint64_t* full = reinterpret_cast<uint64_t*>(sbias + p.bias_floats);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;            // [kNacc]
  uint64_t* tempty = tfull + Cfg::kNacc;  // [kNacc]
  uint64_t* bres_full = tempty + Cfg::kNacc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres_full + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  constexpr uint32_t kMmaWarp = Cfg::kMma;
  int mc_rank = 0;
  if constexpr (CG2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(mc_rank));
  constexpr bool cg2 = CG2;

  if (threadIdx.x == 32 * kMmaWarp + 1) {  // descriptor fetches overlap the prologue
    for (int i = 0; i < p.num_sub; ++i) prefetch_tmap(&p.tmA[i]);
    prefetch_tmap(&p.tmB);
    if (p.store_mode) prefetch_tmap(&p.tmY);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], kProducers);  // every producer arrives once per stage
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < Cfg::kNacc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], cg2 ? 2 * kEpi : 32 * kEpi);  // cg2: one arrive per epilogue warp of the pair
    }
    mbar_init(bres_full, 1);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) {
    if constexpr (cg2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(Cfg::kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(tmem_slot, Cfg::kTmemCols);
      tmem_relinquish();
    }
    if (lane == 0) trace_event(p.trace, TR_PRELOOP);  // TMEM granted (tools/cta_timeline.py)
  }
  if (p.bias_floats) {
    pdl_wait();  // the bias may be produced by the preceding kernel
    for (int i = threadIdx.x; i < p.bias_floats; i += Cfg::kThreadsN) sbias[i] = __ldg(p.bias + i);
  }
  // Piece table (all threads).
  if (p.a_mode != A_TILED) {
    for (int s = 0; s < p.num_sub; ++s) {
      const SubProb& sp = p.sub[s];
      for (int pc = threadIdx.x; pc < sp.num_pieces; pc += Cfg::kThreadsN)
        pieces[sp.piece_begin + pc] = make_piece(p, sp, pc);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (CG2) mc_cluster_sync();  // the peer's barriers exist before any remote arrive / complete_tx
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();

  unsigned long long* trace = (blockIdx.x == 0) ? p.trace : nullptr;
  if (trace && threadIdx.x == 0) trace[1023] = clock64();
  uint64_t t_start = 0;
  if (p.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

  // Whole [b_res_rows, BN] resident panel of this CTA's (group, n-tile), once, issued
  // by the EPILOGUE warps (idle until the first accumulator): a TMA issuer completes
  // its requests one after another (~500 cycles each, tools/tmabw.cu), so panel boxes
  // queued on the producers' threads would delay their first A stage.
  auto issue_bres_panel = [&](int issuer, int nissuers) {
    if (p.b_mode != B_RESIDENT || static_cast<int>(blockIdx.x) >= p.total_tiles) return;
    constexpr int kBChunks = BN / Cfg::kBChunk;
    int s0, mt0, g0, nt0;
    decompose_tile(p, blockIdx.x, s0, mt0, g0, nt0);
    const int col0 = g0 * p.cog + nt0 * BN;
    if (issuer == 0 && elect_one()) mbar_arrive_expect_tx(bres_full, static_cast<uint32_t>(p.b_res_rows) * BN * 2);
    __syncwarp();
    if (elect_one()) {
      if constexpr (GP) {
        // one box of all b_res_rows rows per packed group's 32 columns
        for (int ch = issuer; ch < kBChunks; ch += nissuers)
          tma_load_2d(sB0 + static_cast<size_t>(ch) * p.b_res_rows * Cfg::kBRowBytes, &p.tmB, bres_full,
                      col0 + ch * Cfg::kBChunk, 0);
      } else {
        for (int r = issuer * Cfg::kBRows; r < p.b_res_rows; r += nissuers * Cfg::kBRows)
#pragma unroll
          for (int ch = 0; ch < kBChunks; ++ch)
            tma_load_2d(sB0 + static_cast<size_t>(ch) * p.b_res_rows * Cfg::kBRowBytes +
                            static_cast<size_t>(r) * Cfg::kBRowBytes,
                        &p.tmB, bres_full, col0 + ch * Cfg::kBChunk, r);
      }
    }
    __syncwarp();
  };

  if (warp >= kEpi && warp < kEpi + kProducers) {
    // ------------------------------------------------------------ producers
    // Every producer walks every stage and issues a round-robin share of its
    // TMA requests (pieces j = pw mod 4; B chunks after them), arriving on the
    // stage's full barrier with its own expect_tx. A single issuing thread
    // completes about one request per ~500 cycles (tools/tmabw.cu), so a stage's
    // requests are spread over four issuers.
    const int pw = static_cast<int>(warp) - kEpi;
    const int box = p.a_box_ch;
    const int pps = KS * (kBK / box);  // pieces per stage
    const uint32_t piece_bytes = kBM * box * 2;
    const int a_mode = p.a_mode;
    const int b_mode = p.b_mode;
    constexpr int kBChunks = BN / Cfg::kBChunk;
    constexpr uint32_t kBChunkBytes = Cfg::kBRows * Cfg::kBRowBytes;  // one streamed B box
    // bytes this producer loads per stage (same for every stage)
    uint32_t my_tx = 0;
    for (int j = pw; j < pps; j += kProducers) my_tx += piece_bytes;
    if (b_mode == B_PIECES)
      for (int j = pw; j < pps; j += kProducers) my_tx += kBChunks * box * Cfg::kBRowBytes;
    if (b_mode == B_STREAM && !p.b_kmajor)
      for (int ch = 0; ch < (cg2 ? kBChunks / 2 : kBChunks); ++ch)
        if ((pps + ch) % kProducers == pw) my_tx += kBChunkBytes;
    if constexpr (cg2) my_tx *= 2;  // the leader's barrier receives both CTAs' (identical) shares
    if (b_mode == B_STREAM && p.b_kmajor)
      for (int u = 0; u < KS; ++u)
        if ((pps + u) % kProducers == pw) my_tx += BN * 128;
    // Per-tile producer setup (tile decomposition, im2col base coordinates,
    // split range): divisions and parameter loads that took ~0.9 us after the
    // PDL wait for the first tile (tools/cta_timeline.py). The first tile's is
    // computed before the wait, every next one right after the current tile's
    // last stage is issued.
    struct ProdTile {
      const CUtensorMap* tmA;
      const int4* ptab;
      int a_r, a_c, b_r, b_c, m0, n, cx, cy, cz, col0, npieces, cbase, st0, st1;
    };
    auto prod_setup = [&](int tile) {
      ProdTile t;
      int s, mt, g, nt, ks, z1, z2, lt = mc_tile<CG2>(p, tile);
      split_batch(p, lt, z1, z2);
      decompose_tile(p, lt, s, mt, g, nt, ks);
      t.a_r = batch_row(p.ba, z1, z2);
      t.a_c = batch_col(p.ba, z1, z2);
      t.b_r = batch_row(p.bb, z1, z2);
      t.b_c = batch_col(p.bb, z1, z2);
      const SubProb& sp = p.sub[s];
      t.tmA = &p.tmA[s];
      t.m0 = mt * kBM;
      const int x = t.m0 % sp.gx;
      int rest = t.m0 / sp.gx;
      const int y = rest % sp.gy;
      rest /= sp.gy;
      const int z = rest % sp.gz;
      t.n = rest / sp.gz;
      t.cx = sp.a_lo[0] + x * sp.a_st[0];
      t.cy = sp.a_lo[1] + y * sp.a_st[1];
      t.cz = sp.a_lo[2] + z * sp.a_st[2];
      t.col0 = g * p.cog + nt * BN;
      t.npieces = sp.num_pieces;
      t.cbase = g * p.cig;
      t.ptab = pieces + sp.piece_begin;
      split_range(p, sp.num_stages, ks, t.st0, t.st1);
      return t;
    };
    ProdTile pt{};
    if (static_cast<int>(blockIdx.x) < p.total_tiles) pt = prod_setup(blockIdx.x);
    // Optional: this producer's share of the first stage -> L2 before the wait (a
    // prefetch only moves DRAM latency under the preceding grid's tail; the real
    // loads still come after the wait, and L2 is the point of coherence).
    if (p.l2_prefetch && !cg2 && static_cast<int>(blockIdx.x) < p.total_tiles && elect_one()) {
      const int pc0 = pt.st0 * pps;
      for (int j = pw; j < pps; j += kProducers) {
        const int pc = pc0 + j;
        if (a_mode == A_TILED) {
          tma_prefetch_2d(pt.tmA, pc * kBK + pt.a_c, pt.m0 + pt.a_r);
          continue;
        }
        if (pc >= pt.npieces) break;
        const int4 e = pt.ptab[pc];
        const int c = pt.cbase + e.x;
        const uint16_t ox = static_cast<uint16_t>(e.y & 0xFFFF), oy = static_cast<uint16_t>(e.y >> 16);
        if (a_mode == A_IM2COL4) tma_prefetch_im2col_4d(pt.tmA, c, pt.cx, pt.cy, pt.n, ox, oy);
        else if (a_mode == A_IM2COL3) tma_prefetch_im2col_3d(pt.tmA, c, pt.cx, pt.n, ox);
        else tma_prefetch_im2col_5d(pt.tmA, c, pt.cx, pt.cy, pt.cz, pt.n, ox, oy, static_cast<uint16_t>(e.z));
      }
    }
    __syncwarp();
    // Everything above is parameter arithmetic: it runs before the wait, so
    // the first TMA issues right after the preceding grid's memory is visible.
    pdl_wait();  // operands may be produced by the preceding kernel
    if (warp == kEpi && lane == 0) trace_event(p.trace, TR_PDL_DONE);
    // (a resident B panel is issued by the epilogue warps: issue_bres_panel)
    uint32_t slot = 0, phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x) {
      const int a_r = pt.a_r, a_c = pt.a_c, b_r = pt.b_r, b_c = pt.b_c;
      const CUtensorMap* tmA = pt.tmA;
      const int m0 = pt.m0, n = pt.n, cx = pt.cx, cy = pt.cy, cz = pt.cz;
      const int col0 = pt.col0, npieces = pt.npieces, cbase = pt.cbase;
      const int4* ptab = pt.ptab;
      const int st0 = pt.st0, st1 = pt.st1;
      for (int st = st0; st < st1; ++st, ++it) {
        mbar_wait(&empty[slot], phase ^ 1);
        if (elect_one()) {
          if (trace && pw == 0 && it < 128) trace[2 * it] = clock64();
          if (it == 0 && pw == 0) trace_event(p.trace, TR_FIRST_ISSUE);
          uint8_t* sA = sA0 + slot * Cfg::kABytes;
          uint8_t* sB = sB0 + slot * kBSlotBytes;
          if constexpr (cg2) {
            // both CTAs' loads complete on the leader's barrier; only its producers arrive
            if (mc_rank == 0) mbar_arrive_expect_tx(&full[slot], my_tx);
            const uint32_t lbar = mc_leader_addr(&full[slot]);
            for (int j = pw; j < pps; j += kProducers)
              tma_load_2d_cg2(sA + j * piece_bytes, tmA, lbar, (st * pps + j) * kBK, m0);
#pragma unroll
            for (int ch = 0; ch < kBChunks / 2; ++ch)
              if ((pps + ch) % kProducers == pw)
                tma_load_2d_cg2(sB + ch * kBChunkBytes, &p.tmB, lbar,
                                col0 + mc_rank * (BN / 2) + ch * Cfg::kBChunk, st * Cfg::kBRows);
          } else {
          if (my_tx) mbar_arrive_expect_tx(&full[slot], my_tx);
          else mbar_arrive(&full[slot]);
          for (int j = pw; j < pps; j += kProducers) {
            const int pc = st * pps + j;
            void* dA = sA + j * piece_bytes;
            if (a_mode == A_TILED) {
              tma_load_2d(dA, tmA, &full[slot], pc * kBK + a_c, m0 + a_r);
              continue;
            }
            // Past the last piece: re-read the last real A piece (finite data)
            // against zero B rows (rows >= k_rows are out of bounds -> 0).
            int4 e = ptab[pc < npieces ? pc : npieces - 1];
            if (pc >= npieces) e.w = p.k_rows;
            const int c = cbase + e.x;
            const uint16_t ox = static_cast<uint16_t>(e.y & 0xFFFF);
            const uint16_t oy = static_cast<uint16_t>(e.y >> 16);
            if (a_mode == A_IM2COL4) {
              tma_im2col_4d(dA, tmA, &full[slot], c, cx, cy, n, ox, oy);
            } else if (a_mode == A_IM2COL3) {
              tma_im2col_3d(dA, tmA, &full[slot], c, cx, n, ox);
            } else {
              tma_im2col_5d(dA, tmA, &full[slot], c, cx, cy, cz, n, ox, oy,
                            static_cast<uint16_t>(e.z));
            }
            if (b_mode == B_PIECES) {
#pragma unroll
              for (int ch = 0; ch < kBChunks; ++ch)
                tma_load_2d(sB + ch * kBChunkBytes + j * box * Cfg::kBRowBytes, &p.tmB, &full[slot],
                            col0 + ch * Cfg::kBChunk, e.w);
            }
          }
          if (b_mode == B_STREAM && !p.b_kmajor) {
#pragma unroll
            for (int ch = 0; ch < kBChunks; ++ch)
              if ((pps + ch) % kProducers == pw)
                tma_load_2d(sB + ch * kBChunkBytes, &p.tmB, &full[slot], col0 + ch * Cfg::kBChunk + b_c,
                            st * Cfg::kBRows + b_r);
          } else if (b_mode == B_STREAM) {
            // K-major B: sub-block u = BN rows (N) x 64 K, 128-byte SW128 rows like A
#pragma unroll
            for (int u = 0; u < KS; ++u)
              if ((pps + u) % kProducers == pw)
                tma_load_2d(sB + u * BN * 128, &p.tmB, &full[slot], st * Cfg::kBRows + u * kBK + b_c, col0 + b_r);
          }
          }  // !cg2
          if (trace && pw == 0 && it < 128) trace[2 * it + 1] = clock64();
        }
        __syncwarp();
        if (++slot == static_cast<uint32_t>(S)) {
          slot = 0;
          phase ^= 1;
        }
      }
      if (tile + static_cast<int>(gridDim.x) < p.total_tiles) pt = prod_setup(tile + gridDim.x);
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // Descriptor templates; per stage/k only the 14-bit start-address field
    // (bits 0-13, address >> 4) changes, so plain 64-bit adds update it.
    uint32_t a_layout, a_sbo, a_lbo;
    uint32_t a_koff[4];  // byte offset of k-step k within a 64-deep A sub-block
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
    const uint32_t b_lbo = b_res ? p.b_res_rows * Cfg::kBRowBytes : Cfg::kBRows * Cfg::kBRowBytes;
    const bool bkm = p.b_kmajor != 0;
    const uint64_t bdesc0 = bkm ? smem_desc(smem_u32(sB0), 16, 1024, 2)
                                : smem_desc(smem_u32(sB0), b_lbo, 8 * Cfg::kBRowBytes, Cfg::kBLayout);
    // per k-step / per 64-deep sub-block descriptor advances (16-byte units)
    const uint32_t kBk = bkm ? 2u : (16 * Cfg::kBRowBytes) >> 4;
    const uint32_t kBsub = bkm ? static_cast<uint32_t>(BN * 128) >> 4 : (kBK * Cfg::kBRowBytes) >> 4;
    const uint32_t idesc = bkm ? idesc_f16_f32(kBM, BN, 0, 0) : Cfg::kIdesc;
    constexpr uint32_t kBst = (Cfg::kBRows * Cfg::kBRowBytes) >> 4;  // per stage (resident)
    constexpr uint32_t kBslot = kBSlotBytes >> 4;                    // per ring slot
    constexpr uint32_t kAslot = Cfg::kABytes >> 4;
    constexpr uint32_t kAsub = Cfg::kSubA >> 4;
    if (b_res && static_cast<int>(blockIdx.x) < p.total_tiles) {
      mbar_wait(bres_full, 0);
      tc_fence_after();
    }
    uint32_t slot = 0, phase = 0, acc = 0, acc_phase = 0;
    int it = 0;
    const uint32_t idesc_mma = cg2 ? idesc_f16_f32(2 * kBM, BN, 0, 1) : idesc;
    // cg2: the leader issues every MMA of the pair; the peer's MMA warp idles
    for (int tile = blockIdx.x + ((cg2 && mc_rank) ? p.total_tiles : 0); tile < p.total_tiles;
         tile += gridDim.x) {
      int s, mt, g, nt, ks, z1, z2, lt = mc_tile<CG2>(p, tile);
      split_batch(p, lt, z1, z2);
      decompose_tile(p, lt, s, mt, g, nt, ks);
      int st0, st1;
      split_range(p, p.sub[s].num_stages, ks, st0, st1);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (int st = st0; st < st1; ++st, ++it) {
        mbar_wait(&full[slot], phase);
        tc_fence_after();
        if (it == 0 && lane == 0) trace_event(p.trace, TR_FIRST_FULL);
        if (trace && lane == 0 && it < 128) trace[256 + 2 * it] = clock64();
        const uint64_t a = adesc0 + slot * kAslot;
        const uint64_t b = bdesc0 + (b_res ? st * kBst : slot * kBslot);
        if (elect_one()) {
          if constexpr (GP) {
            // sub-block u = tap st*KS + u (one 64-channel piece); K16 step k of it is
            // packed group k / kpg's step k % kpg; its B rows are that group's
            // [tap*cig + 16*(k % kpg), +16) of its own 32-column chunk
            const int kpg = p.gp_kpg;
            const uint32_t kBgrp = static_cast<uint32_t>(p.b_res_rows * Cfg::kBRowBytes) >> 4;
#pragma unroll
            for (int u = 0; u < KS; ++u) {
              const int t = st * KS + u;
              if (t >= p.gp_taps) continue;  // K padding of the last stage
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k) {
                const int q = kpg == 1 ? k : k >> 1, kk = k - q * kpg;
                const uint32_t brow = static_cast<uint32_t>((t * kpg + kk) * 16);
                umma_f16(tmem_d + q * 32, a + u * kAsub + (a_koff[k] >> 4),
                         bdesc0 + q * kBgrp + ((brow * Cfg::kBRowBytes) >> 4), Cfg::kIdesc,
                         (st != st0 || u != 0 || kk != 0) ? 1u : 0u);
              }
            }
          } else {
#pragma unroll
          for (int u = 0; u < KS; ++u)
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              if constexpr (cg2)
                umma_f16_cg2(tmem_d, a + u * kAsub + (a_koff[k] >> 4), b + u * kBsub + k * kBk, idesc_mma,
                             ((st - st0) | u | k) != 0);
              else
                umma_f16(tmem_d, a + u * kAsub + (a_koff[k] >> 4), b + u * kBsub + k * kBk,
                         idesc, ((st - st0) | u | k) != 0);
            }
          }  // !GP
          if constexpr (cg2) umma_commit_cg2(&empty[slot]);
          else umma_commit(&empty[slot]);
        }
        __syncwarp();
        if (trace && lane == 0 && it < 128) trace[256 + 2 * it + 1] = clock64();
        if (++slot == static_cast<uint32_t>(S)) {
          slot = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) {
        if constexpr (cg2) umma_commit_cg2(&tfull[acc]);
        else umma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++acc == static_cast<uint32_t>(Cfg::kNacc)) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp < kEpi) {
    // ------------------------------------------------------------ epilogue
    pdl_wait();  // Y / Yin may be in use by the preceding kernel (and W by the panel load)
    issue_bres_panel(static_cast<int>(warp), kEpi);
    const uint32_t q = warp & 3, hh = warp >> 2;
    constexpr int kHs = kEpi / 4;  // column chunks are dealt round-robin over the kHs warps of a quadrant
    uint8_t* wbuf = epi_smem + warp * Cfg::kEpiWarpBytes;
    uint32_t acc = 0, acc_phase = 0, chunk = 0;
    if (p.ksplit > 1) {
      // Split-K partial: the CTA's one tile (grid == total_tiles) goes from TMEM
      // to a padded [128][BN + 4] fp32 image over the drained operand ring (every
      // MMA, hence every operand read, completed before tfull); cluster_reduce
      // below combines the ksplit partials of the cluster in a fixed order.
      float* part = reinterpret_cast<float*>(smem);
      constexpr int kChunk = BN < 32 ? BN : 32;
      split_row_offsets<BN>(p, reinterpret_cast<int64_t*>(epi_smem), threadIdx.x, 32 * kEpi);
      for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (threadIdx.x == 0) trace_event(p.trace, TR_FIRST_TFULL);
#pragma unroll 1
        for (int c0 = static_cast<int>(hh) * kChunk; c0 < BN; c0 += kHs * kChunk) {
          uint32_t r[32];
          const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * BN + c0;
          if (kChunk == 32) tmem_ld_32x32b_x32(taddr, r);
          else tmem_ld_32x32b_x16(taddr, r);
          tmem_ld_wait();
          float4* dst = reinterpret_cast<float4*>(part + (q * 32 + lane) * (BN + 4) + c0);
#pragma unroll
          for (int i = 0; i < kChunk / 4; ++i)
            dst[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                 __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        if (threadIdx.x == 0) trace_x(p.trace, 4);
      }
    } else if (p.store_mode) {
      // TMA store: thread = tile row (tcgen05.ld 32x32b); each warp stages its
      // 32 rows x cw columns (SW128 / SW64 swizzled, conflict-free) and issues
      // one bulk tensor store (or reduce-add for accumulate) per chunk; two
      // staging buffers per warp. fp16 outputs with BN >= 64 stage 64 columns
      // (two 32-column TMEM loads) as 128-byte rows: the store engine is
      // request-bound, and 4 KB requests double the bytes per request of the
      // 2 KB ones (1x1 convs / expansion GEMMs are epilogue-bound).
      // Row-linear outputs only (GMM, forward conv).
      // Epilogue operands are fetched ahead of their use (measured: a bias load
      // issued next to its add costs ~1000 cycles per 32 columns under the
      // store traffic): the tile's bias is loaded before the accumulator wait,
      // one column per lane (then broadcast with shuffles), and the residual of
      // the next 32 columns is in flight while the current ones are processed.
      const int cw = p.epi_cw;  // 32, or 64 for fp16 output
      const int line_bytes = cw * (p.out_f16 ? 2 : 4);
      const bool epi_on = p.bias || p.relu || p.residual;
      int local = 0;
      for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x, ++local) {
        int s, mt, g, nt, z1, z2, lt = mc_tile<CG2>(p, tile);
        split_batch(p, lt, z1, z2);
        decompose_tile(p, lt, s, mt, g, nt);
        const int c_r = batch_row(p.bc, z1, z2), c_c = batch_col(p.bc, z1, z2);
        const int64_t row_local = static_cast<int64_t>(mt) * kBM + q * 32 + lane;
        const int64_t row = row_local + c_r;  // row of the C tensor
        const int64_t colb_tile = static_cast<int64_t>(g) * p.cog + nt * BN;  // bias column (per problem)
        const int64_t col_tile = colb_tile + c_c;                               // column of the C tensor
        const int valid_tile = p.cog - nt * BN;  // columns of this tile inside the group
        // bias of the next 32 columns, one column per lane (prefetched a chunk ahead)
        const int c_first = static_cast<int>(hh) * cw;  // this warp's first chunk
        float bnext = (p.bias && c_first + static_cast<int>(lane) < valid_tile)
                          ? __ldg(p.bias + colb_tile + c_first + lane) : 0.0f;
        // residual rows past M are clipped by the TMA store and never read
        const uint16_t* res_row = (p.residual && row_local < p.sub[0].m_count)
                                      ? p.residual + row * p.ldy + col_tile : nullptr;
        uint4 rp[4];  // fp16 residual of the next 32 columns
        auto fetch_res = [&](int c) {
          if (res_row && valid_tile - c >= 32 && (reinterpret_cast<uintptr_t>(res_row + c) & 15) == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) rp[i] = __ldg(reinterpret_cast<const uint4*>(res_row + c) + i);
          }
        };
        fetch_res(c_first);
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (local == 0 && threadIdx.x == 0) trace_event(p.trace, TR_FIRST_TFULL);
        if (trace && threadIdx.x == 0 && local < 64) trace[512 + 2 * local] = clock64();
#pragma unroll 1
        for (int c0 = c_first; c0 < BN; c0 += kHs * cw, ++chunk) {
          if (c0 >= valid_tile) continue;  // warp-uniform: chunk past the group
          uint8_t* buf = wbuf + (chunk & 1) * 4096;
          uint8_t* dst = buf + lane * line_bytes;
          __syncwarp();  // lane 0 has retired the store that last read `buf`
#pragma unroll 1
          for (int h = 0; h < cw; h += 32) {
            uint32_t r[32];
            const int cc = c0 + h;
            const int next_cc = h + 32 < cw ? cc + 32 : c0 + kHs * cw;  // this warp's next 32 columns
            tmem_ld_32x32b_x32(tmem_base + ((q * 32u) << 16) + acc * BN + cc, r);
            tmem_ld_wait();
            const int lim = valid_tile - cc;
            if (lim <= 0) break;  // warp-uniform: half past the group (TMA clips it)
            if (epi_on) {
              float* v = reinterpret_cast<float*>(r);
              // C-ABI order: + bias, + residual, activation
              if (p.bias && p.bias_floats && lim >= 32) {
                // staged bias: eight 16-byte shared-memory broadcasts per 32 columns
                const float4* b4 = reinterpret_cast<const float4*>(sbias + colb_tile + cc);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const float4 b = b4[i];
                  v[4 * i] += b.x; v[4 * i + 1] += b.y; v[4 * i + 2] += b.z; v[4 * i + 3] += b.w;
                }
              } else if (p.bias) {
                const float bcur = bnext;
                const int nc = next_cc + static_cast<int>(lane);
                bnext = nc < valid_tile ? __ldg(p.bias + colb_tile + nc) : 0.0f;
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += __shfl_sync(0xffffffffu, bcur, i);
              }
              if (res_row) {
                if (lim >= 32 && (reinterpret_cast<uintptr_t>(res_row + cc) & 15) == 0) {
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const __half2* hv = reinterpret_cast<const __half2*>(&rp[i]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                      const float2 f = __half22float2(hv[j]);
                      v[8 * i + 2 * j] += f.x;
                      v[8 * i + 2 * j + 1] += f.y;
                    }
                  }
                } else {
#pragma unroll
                  for (int i = 0; i < 32; ++i)
                    if (i < lim)
                      v[i] += __half2float(__ushort_as_half(
                          __ldg(reinterpret_cast<const unsigned short*>(res_row + cc) + i)));
                }
                fetch_res(next_cc);  // in flight during this chunk's conversion and store
              }
              epi_act_n<32>(v, p.relu);
            }
            if (p.out_f16) {
              const int hp = h >> 3;  // first 16-byte piece of this half (0 or 4)
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                uint4 u;
                __half2 h0 = __floats2half2_rn(__uint_as_float(r[8 * c]), __uint_as_float(r[8 * c + 1]));
                __half2 h1 = __floats2half2_rn(__uint_as_float(r[8 * c + 2]), __uint_as_float(r[8 * c + 3]));
                __half2 h2 = __floats2half2_rn(__uint_as_float(r[8 * c + 4]), __uint_as_float(r[8 * c + 5]));
                __half2 h3 = __floats2half2_rn(__uint_as_float(r[8 * c + 6]), __uint_as_float(r[8 * c + 7]));
                u.x = *reinterpret_cast<uint32_t*>(&h0);
                u.y = *reinterpret_cast<uint32_t*>(&h1);
                u.z = *reinterpret_cast<uint32_t*>(&h2);
                u.w = *reinterpret_cast<uint32_t*>(&h3);
                const int piece = cw == 64 ? ((hp + c) ^ (lane & 7))          // SW128
                                           : (c ^ ((lane >> 1) & 3));         // SW64
                *reinterpret_cast<uint4*>(dst + (piece << 4)) = u;
              }
            } else {
#pragma unroll
              for (int c = 0; c < 8; ++c)
                *reinterpret_cast<uint4*>(dst + ((c ^ (lane & 7)) << 4)) =
                    make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);  // SW128
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int col = static_cast<int>(col_tile) + c0;
            const int row0 = mt * kBM + static_cast<int>(q) * 32 + c_r;
            if (p.store_mode == 2) tma_reduce_add_2d(&p.tmY, buf, col, row0);
            else tma_store_2d(&p.tmY, buf, col, row0);
            tma_store_commit();
            tma_store_wait_read<1>();
          }
        }
        if (trace && threadIdx.x == 0 && local < 64) trace[513 + 2 * local] = clock64();
        tc_fence_before();
        if constexpr (cg2) {  // one arrive per warp on the leader's barrier
          __syncwarp();
          if (lane == 0) {
            if (mc_rank == 0) mbar_arrive(&tempty[acc]);
            else mbar_arrive_rank0(&tempty[acc]);
          }
        } else {
          mbar_arrive(&tempty[acc]);
        }
        if (++acc == static_cast<uint32_t>(Cfg::kNacc)) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (lane == 0) tma_store_wait_read<0>();  // smem reads done; the grid end flushes the writes
      if (threadIdx.x == 0 && p.trace) {
        tma_store_wait_all<0>();  // (trace only) the stores themselves complete
        trace_event(p.trace, TR_STORES_DONE);
      }
    } else {
      // Generic: TMEM -> registers (thread = output row) -> smem transpose ->
      // coalesced stores of 32-column row segments at per-row output offsets
      // (T2D scatters class rows to strided output pixels).
      float* stg = reinterpret_cast<float*>(wbuf);          // 32 x 36 fp32
      int64_t* row_off = reinterpret_cast<int64_t*>(wbuf + 32 * 36 * 4);
      const bool vec_ok = (p.ldy % 8 == 0) && (p.cog % 8 == 0) &&
                          ((reinterpret_cast<uintptr_t>(p.Y) & 15) == 0) &&
                          (!p.accumulate || (reinterpret_cast<uintptr_t>(p.Yin) & 15) == 0);
      int local = 0;
      for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x, ++local) {
        int s, mt, g, nt;
        decompose_tile(p, mc_tile<CG2>(p, tile), s, mt, g, nt);
        const SubProb& sp = p.sub[s];
        {
          const int m = mt * kBM + static_cast<int>(q * 32 + lane);
          int64_t off = -1;
          if (m < sp.m_count) {
            int x = m % sp.gx, rest = m / sp.gx;
            int y = rest % sp.gy;
            rest /= sp.gy;
            int z = rest % sp.gz;
            int n = rest / sp.gz;
            const int ox = x * sp.o_st[0] + sp.o_b[0];
            const int oy = y * sp.o_st[1] + sp.o_b[1];
            const int oz = z * sp.o_st[2] + sp.o_b[2];
            const int64_t pix = ((static_cast<int64_t>(n) * p.out_dims[2] + oz) * p.out_dims[1] + oy) *
                                    p.out_dims[0] + ox;
            off = pix * p.ldy + g * p.cog + nt * BN;
          }
          row_off[lane] = off;
        }
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (trace && threadIdx.x == 0 && local < 64) trace[512 + 2 * local] = clock64();
        if (local == 0 && threadIdx.x == 0) trace_event(p.trace, TR_FIRST_TFULL);
        const int ncol0 = nt * BN;
        constexpr int kChunk = BN < 32 ? BN : 32;
        constexpr int kLanesPerRow = kChunk / 4;
        constexpr int kRowsPerPass = 32 / kLanesPerRow;
#pragma unroll 1
        for (int c0 = static_cast<int>(hh) * kChunk; c0 < BN; c0 += kHs * kChunk) {
          uint32_t r[32];
          const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * BN + c0;
          if (kChunk == 32) tmem_ld_32x32b_x32(taddr, r);
          else tmem_ld_32x32b_x16(taddr, r);
          tmem_ld_wait();
          const int valid = min(kChunk, p.cog - (ncol0 + c0));
          if (valid <= 0) continue;  // warp-uniform
          __syncwarp();
          float* my = stg + lane * 36;
#pragma unroll
          for (int i = 0; i < kChunk; i += 4)
            *reinterpret_cast<float4*>(my + i) = make_float4(
                __uint_as_float(r[i]), __uint_as_float(r[i + 1]), __uint_as_float(r[i + 2]),
                __uint_as_float(r[i + 3]));
          __syncwarp();
          const int col = (lane % kLanesPerRow) * 4;
#pragma unroll 4
          for (int rr = lane / kLanesPerRow; rr < 32; rr += kRowsPerPass) {
            const int64_t ro = row_off[rr];
            if (ro < 0 || col >= valid) continue;
            const int64_t off = ro + c0 + col;
            float4 v = *reinterpret_cast<const float4*>(stg + rr * 36 + col);
            const bool vec = vec_ok && col + 4 <= valid;
            if (p.accumulate) {
              if (vec) {
                const float4 t = *reinterpret_cast<const float4*>(p.Yin + off);
                v.x = t.x + v.x; v.y = t.y + v.y; v.z = t.z + v.z; v.w = t.w + v.w;
              } else {
                float* vv = reinterpret_cast<float*>(&v);
                for (int i = 0; i < 4 && col + i < valid; ++i) vv[i] = p.Yin[off + i] + vv[i];
              }
            }
            if (p.bias || p.relu || p.residual) {
              const int64_t colb = g * p.cog + ncol0 + c0 + col;
              epi_run<4>(reinterpret_cast<float*>(&v), p.bias, colb, valid - col,
                         p.residual ? p.residual + off : nullptr, p.relu);
            }
            if (p.out_f16) {
              __half* y = reinterpret_cast<__half*>(p.Y) + off;
              if (vec) {
                __half2 h0 = __floats2half2_rn(v.x, v.y), h1 = __floats2half2_rn(v.z, v.w);
                uint2 u;
                u.x = *reinterpret_cast<uint32_t*>(&h0);
                u.y = *reinterpret_cast<uint32_t*>(&h1);
                *reinterpret_cast<uint2*>(y) = u;
              } else {
                const float* vv = reinterpret_cast<const float*>(&v);
                for (int i = 0; i < 4 && col + i < valid; ++i) y[i] = __float2half_rn(vv[i]);
              }
            } else {
              float* y = reinterpret_cast<float*>(p.Y) + off;
              if (vec) {
                *reinterpret_cast<float4*>(y) = v;
              } else {
                const float* vv = reinterpret_cast<const float*>(&v);
                for (int i = 0; i < 4 && col + i < valid; ++i) y[i] = vv[i];
              }
            }
          }
          __syncwarp();
        }
        if (trace && threadIdx.x == 0 && local < 64) trace[513 + 2 * local] = clock64();
        tc_fence_before();
        if constexpr (cg2) {  // one arrive per warp on the leader's barrier
          __syncwarp();
          if (lane == 0) {
            if (mc_rank == 0) mbar_arrive(&tempty[acc]);
            else mbar_arrive_rank0(&tempty[acc]);
          }
        } else {
          mbar_arrive(&tempty[acc]);
        }
        if (++acc == static_cast<uint32_t>(Cfg::kNacc)) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) trace_x(p.trace, 5);
  if constexpr (cg2) mc_cluster_sync();  // the leader's MMAs into this CTA's TMEM are done
  if (p.ksplit > 1) cluster_reduce<BN>(p, reinterpret_cast<const float*>(smem), reinterpret_cast<int64_t*>(epi_smem));
  if (warp == kMmaWarp) {
    if constexpr (cg2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Cfg::kTmemCols)
                   : "memory");
    else
      tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
  if (threadIdx.x == 0) trace_event(p.trace, TR_EXIT);
  if (p.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
    uint64_t t_end;
    uint32_t smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[2048 + 4 * blockIdx.x] = t_start;
    p.trace[2048 + 4 * blockIdx.x + 1] = t_end;
    p.trace[2048 + 4 * blockIdx.x + 2] = smid;
    p.trace[2048 + 4 * blockIdx.x + 3] = (p.total_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  }
}

}  // namespace tb
