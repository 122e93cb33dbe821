// halo.cuh — direct (halo-tile) tcgen05 convolution for stride-1 convs
// (C2D 3x3 s1, the BASELINE headline; any KH x KW, dilation, padding, groups).
//
// Why a second conv kernel: im2col re-reads each input pixel once per tap
// through L2 (9x for 3x3) and needs one TMA request + one barrier round per
// 64-deep K slab. Measured on B200 (tools/tmabw.cu, tools/trace_igemm.py) each
// TMA issuer completes ~1 request per ~500 cycles and a barrier/MMA round costs
// ~450 cycles of single-warp latency — more than the math of a 128x64x64 slab.
//
// Here a tile is R output rows x Wt output columns of one image. Its input
// footprint — (R + (KH-1)d) padded input rows x Wv = Wt + (KW-1)d columns x 64
// channels — is ONE tiled TMA box (zero fill supplies the padding) into smem,
// laid out as "virtual pixels" v = r*Wv + c with 128-byte SW128 rows. For tap
// (ty, tx) the UMMA A operand is simply the 128 rows starting at
// v0 = ty*d*Wv + tx*d: a descriptor start-address offset (the hardware swizzles
// on absolute smem address bits; tools/umma_probe.cu verifies any 128-byte row
// start is exact with base_offset = 0). Output virtual pixel m of the tile is
// (m / Wv, m % Wv); columns >= Wt and rows >= R are computed and discarded.
// All KH*KW taps x 4 K-steps are issued per barrier round (36 MMAs for 3x3),
// weights stay resident in smem, so per tile the CTA moves one input slab in
// and one output tile out.
//
// Reduction order differs from the reference's (rh, rw, rc) loop only by fp32
// reassociation inside the tensor core; on the reference input distribution
// every partial sum is exact, so results are bit-identical (tests/test_gpu_parity.py).
#pragma once

#include "ptx.cuh"

namespace tb {

constexpr int kHaloThreads = 320;  // warps 0-7 epilogue, 8 producer, 9 MMA
constexpr int kHaloMaxRows = 640;  // smem rows per halo slab (128 B each)

struct alignas(64) HaloParams {
  CUtensorMap tmX;  // 4-D tiled over X[N, H, W, C]: box {64 ch, Wv, HR, 1}, SW128
  CUtensorMap tmW;  // 2-D over W[taps*CIg, CO]: box {min(BN,64), b_box_rows}
  CUtensorMap tmY;  // 4-D over Y[N, OH, OW, CO]: box {32, Wt, R, 1} (store_mode != 0)
  int32_t n, oh, ow, co, cig, cog, groups;
  int32_t kh, kw, dil, pad_h, pad_w;
  int32_t R, Wt, Wv, HR;      // tile rows, tile cols, virtual row width, halo rows
  int32_t tiles_w, tiles_h;   // tiles per image along W / H
  int32_t tiles_n;            // N tiles per group
  int32_t total_tiles;
  int32_t cblocks;            // cig / 64: halo slabs (K stages) per tile
  int32_t b_rows;             // resident weight rows (taps * cig)
  int32_t b_box_rows;         // rows per weight TMA box (divides b_rows, <= 256)
  int32_t stages;             // halo ring depth
  int32_t slab_rows;          // smem rows per slab (>= max tap offset + 128)
  int32_t accumulate, out_f16;
  const float* bias;  // fused epilogue: per-output-column bias (nullable)
  int32_t relu;       // fused epilogue activation (1 ReLU, 2 ReLU6, 3 GELU)
  const uint16_t* residual;  // fused epilogue: fp16 residual in Y's layout (store_mode 0 only)
  int32_t store_mode;         // 0: direct register stores, 1: TMA store, 2: TMA reduce-add (Y += )
  int32_t nacc;               // TMEM accumulator buffers (MMA runs nacc-1 tiles ahead)
  int32_t stage_bytes;        // TMA-store staging buffer bytes (one of two)
  void* Y;
  const float* Yin;
  unsigned long long* trace;
  int32_t l2_prefetch;  // first tile -> L2 before griddepcontrol.wait (ptx.cuh tma_prefetch_*)
};

template <int BN>
struct HaloCfg {
  static constexpr int kBChunk = BN < 64 ? BN : 64;
  static constexpr int kBRowBytes = kBChunk * 2;
  static constexpr uint32_t kBLayout = kBRowBytes == 128 ? 2u : kBRowBytes == 64 ? 4u : 6u;
  static constexpr int kN = BN;  // MMA N (accumulator columns per tile)
  static constexpr uint32_t kIdesc = idesc_f16_f32(128, kN, 0, 1);
  static constexpr int kNacc = (4 * kN <= 512) ? 4 : 2;   // accumulator buffers
  static constexpr int kTmemCols = (kNacc * kN <= 32) ? 32 : (kNacc * kN <= 64) ? 64
                                   : (kNacc * kN <= 128) ? 128 : (kNacc * kN <= 256) ? 256 : 512;
  static size_t smem_bytes(int stages, int slab_rows, int b_rows, int stage_bytes) {
    return 1024 + static_cast<size_t>(stages) * slab_rows * 128 +
           static_cast<size_t>(b_rows) * BN * 2 + 2 * static_cast<size_t>(stage_bytes) + 256;
  }
};

template <int BN, int KH, int KW>  // KH = KW = 0: runtime kernel extents
__global__ void __launch_bounds__(kHaloThreads, 1) conv_halo_kernel(const __grid_constant__ HaloParams p) {
  using Cfg = HaloCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int S = p.stages;
  const uint32_t slab_bytes = static_cast<uint32_t>(p.slab_rows) * 128;
  uint8_t* sA0 = smem;
  uint8_t* sB = smem + static_cast<size_t>(S) * slab_bytes;
  uint8_t* epi = sB + static_cast<size_t>(p.b_rows) * BN * 2;  // 1024-aligned (host)
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + 2 * p.stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;           // [kNacc]
  uint64_t* tempty = tfull + Cfg::kNacc;  // [kNacc]
  uint64_t* bfull = tempty + Cfg::kNacc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  if (threadIdx.x == 0) trace_event(p.trace, TR_ENTRY);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 32 * 8 + 1) {  // descriptor fetches overlap the prologue
    prefetch_tmap(&p.tmX);
    prefetch_tmap(&p.tmW);
    if (p.store_mode == 1 || p.store_mode == 2) prefetch_tmap(&p.tmY);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < Cfg::kNacc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], p.store_mode ? 128 : 256);  // TMA-store modes use warps 0-3; mode 0 all 8
    }
    mbar_init(bfull, 1);
    fence_barrier_init();
  }
  if (warp == 9) {
    tmem_alloc(tmem_slot, Cfg::kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  unsigned long long* trace = (blockIdx.x == 0) ? p.trace : nullptr;
  if (trace && threadIdx.x == 0) trace[1023] = clock64();
  uint64_t t_start = 0;
  if (p.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int tiles_img = p.tiles_h * p.tiles_w;
  const int per_img = tiles_img * p.groups * p.tiles_n;
  // tile -> (n, th, tw, g, nt), n-tile fastest so neighbours share the input slab in L2
  auto decompose = [&](int tile, int& n, int& th, int& tw, int& g, int& nt) {
    nt = tile % p.tiles_n;
    int r = tile / p.tiles_n;
    g = r % p.groups;
    r /= p.groups;
    tw = r % p.tiles_w;
    r /= p.tiles_w;
    th = r % p.tiles_h;
    n = r / p.tiles_h;
  };
  (void)per_img;

  if (warp == 8) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      if (p.l2_prefetch && static_cast<int>(blockIdx.x) < p.total_tiles) {
        // first tile's slabs and the weight panel -> L2 before the wait (ptx.cuh tma_prefetch_*)
        int n, th, tw, g, nt;
        decompose(blockIdx.x, n, th, tw, g, nt);
        for (int cb = 0; cb < p.cblocks && cb < S; ++cb)
          tma_prefetch_4d(&p.tmX, g * p.cig + cb * 64, tw * p.Wt - p.pad_w, th * p.R - p.pad_h, n);
        // The weight panel is shared by every CTA of the (group, n-tile): each CTA
        // prefetches one box of it (l2_prefetch == 2; 1 = every box, measured
        // 0.4 us slower: an SM's TMA unit works through its prefetches in order,
        // ahead of the first real load).
        int box = 0;
        for (int r = 0; r < p.b_rows; r += p.b_box_rows)
          for (int ch = 0; ch < BN / Cfg::kBChunk; ++ch, ++box)
            if (p.l2_prefetch == 1 || box == static_cast<int>(blockIdx.x) / (p.groups * p.tiles_n))
              tma_prefetch_2d(&p.tmW, g * p.cog + nt * BN + ch * Cfg::kBChunk, r);
      }
      // the first tile's coordinates and every loop constant in registers before the
      // wait (parameter loads after it miss the constant cache on the critical path)
      const uint32_t slab_tx = static_cast<uint32_t>(pin(p.HR * p.Wv * 128));
      const int R = pin(p.R), Wt = pin(p.Wt), pad_h = pin(p.pad_h), pad_w = pin(p.pad_w);
      const int cblocks = pin(p.cblocks), cig = pin(p.cig), total = pin(p.total_tiles);
      uint32_t slot = 0, phase = 0;
      int it = 0;
      bool weights_pending = static_cast<int>(blockIdx.x) < total;
      int n, th, tw, g, nt;
      decompose(blockIdx.x, n, th, tw, g, nt);
      n = pin(n), th = pin(th), tw = pin(tw), g = pin(g);
      pdl_wait();  // X / W may be produced by the preceding kernel
      trace_event(p.trace, TR_PDL_DONE);
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        if (tile != static_cast<int>(blockIdx.x)) decompose(tile, n, th, tw, g, nt);
        const int y0 = th * R - pad_h;
        const int x0 = tw * Wt - pad_w;
        for (int cb = 0; cb < cblocks; ++cb, ++it) {
          if (it == 0) trace_event(p.trace, TR_PRELOOP);
          mbar_wait(&empty[slot], phase ^ 1);
          if (trace && it < 128) trace[2 * it] = clock64();
          if (it == 0) trace_event(p.trace, TR_FIRST_ISSUE);
          mbar_arrive_expect_tx(&full[slot], slab_tx);
          tma_load_4d(sA0 + slot * slab_bytes, &p.tmX, &full[slot], g * cig + cb * 64, x0, y0, n);
          if (trace && it < 128) trace[2 * it + 1] = clock64();
          if (weights_pending) {
            // Resident weights of this CTA's (group, n-tile) — grid % (groups*tiles_n)
            // == 0, so every tile of the CTA uses the same panel. Issued after the
            // first slab so the first MMA is not queued behind them; boxes of up to
            // 256 rows that tile b_rows exactly (a box never writes past the panel).
            weights_pending = false;
            const int col0 = g * p.cog + nt * BN;
            mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(p.b_rows) * BN * 2);
            for (int r = 0; r < p.b_rows; r += p.b_box_rows)
#pragma unroll
              for (int ch = 0; ch < BN / Cfg::kBChunk; ++ch)
                tma_load_2d(sB + static_cast<size_t>(ch) * p.b_rows * Cfg::kBRowBytes +
                                static_cast<size_t>(r) * Cfg::kBRowBytes,
                            &p.tmW, bfull, col0 + ch * Cfg::kBChunk, r);
          }
          if (++slot == static_cast<uint32_t>(S)) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    const uint64_t a0 = smem_desc(smem_u32(sA0), 16, 1024, 2);
    const uint64_t b0 = smem_desc(smem_u32(sB), p.b_rows * Cfg::kBRowBytes,
                                  8 * Cfg::kBRowBytes, Cfg::kBLayout);
    const uint32_t slab16 = slab_bytes >> 4;
    // descriptor start-address units (16 B): one virtual pixel row = 128 B = 8
    const int wv_dil = p.Wv * p.dil * 8;   // +1 tap row
    const int dil8 = p.dil * 8;            // +1 tap column
    const int cig_b = (p.cig * Cfg::kBRowBytes) >> 4;  // weight rows of one tap
    constexpr uint32_t kBk16 = (16 * Cfg::kBRowBytes) >> 4;
    const int taps = p.kh * p.kw;
    if (static_cast<int>(blockIdx.x) < p.total_tiles) {
      mbar_wait(bfull, 0);
      tc_fence_after();
      if (trace && lane == 0) trace[1022] = clock64();
    }
    // Flattened stage loop (stage = (tile, channel block)). The barriers of
    // stage i+1 are waited on after all but the last tap of stage i is issued,
    // while the tensor pipe still holds queued MMAs, so the pipe does not drain
    // between stages or tiles.
    const int my_tiles = static_cast<int>(blockIdx.x) < p.total_tiles
                             ? (p.total_tiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                             : 0;
    const int nstage = my_tiles * p.cblocks;
    uint32_t slot = 0, phase = 0, acc = 0, acc_phase = 0;
    auto wait_stage = [&](int i, uint32_t sl, uint32_t ph, uint32_t ac, uint32_t acph) {
      if (i % p.cblocks == 0) mbar_wait(&tempty[ac], acph ^ 1);
      mbar_wait(&full[sl], ph);
      tc_fence_after();
      if (i == 0 && lane == 0) trace_event(p.trace, TR_FIRST_FULL);
    };
    if (nstage > 0) wait_stage(0, 0, 0, 0, 0);
    for (int i = 0; i < nstage; ++i) {
      const int cb = i % p.cblocks;
      const bool last_cb = cb == p.cblocks - 1;
      const uint32_t tmem_d = tmem_base + acc * Cfg::kN;
      // next stage's ring positions
      uint32_t nslot = slot + 1, nphase = phase, nacc = acc, nacc_phase = acc_phase;
      if (nslot == static_cast<uint32_t>(S)) { nslot = 0; nphase ^= 1; }
      if (last_cb && ++nacc == static_cast<uint32_t>(Cfg::kNacc)) { nacc = 0; nacc_phase ^= 1; }
      if (trace && lane == 0 && i < 128) trace[256 + 2 * i] = clock64();
      const uint64_t a_slab = a0 + slot * slab16;
      const uint64_t b_cb = b0 + ((static_cast<uint32_t>(cb * 64) * Cfg::kBRowBytes) >> 4);
      auto issue_tap = [&](int ty, int tx, int t) {
        const uint64_t a = a_slab + static_cast<uint32_t>(ty * wv_dil + tx * dil8);
        const uint64_t b = b_cb + static_cast<uint32_t>(t * cig_b);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_f16(tmem_d, a + 2u * k, b + k * kBk16, Cfg::kIdesc, (cb | t | k) != 0);
      };
      const bool leader = elect_one();
      if constexpr (KH > 0) {
        if (leader) {
#pragma unroll
          for (int t = 0; t < KH * KW - 1; ++t) issue_tap(t / KW, t % KW, t);
        }
      } else {
        if (leader) {
          for (int t = 0; t < taps - 1; ++t) issue_tap(t / p.kw, t % p.kw, t);
        }
      }
      __syncwarp();
      if (i + 1 < nstage) wait_stage(i + 1, nslot, nphase, nacc, nacc_phase);
      if (leader) {
        const int t = taps - 1;
        issue_tap(t / p.kw, t % p.kw, t);
        umma_commit(&empty[slot]);
        if (last_cb) umma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (trace && lane == 0 && i < 128) trace[256 + 2 * i + 1] = clock64();
      slot = nslot; phase = nphase; acc = nacc; acc_phase = nacc_phase;
    }
  } else if (p.store_mode) {
    // ------------------------------------------------------------ epilogue, TMA store
    // Warps 0-3 (TMEM lane quadrants; warps 4-7 idle): tcgen05.ld 32x32b (thread =
    // tile row = virtual pixel) -> the pixel's 32-channel line of a dense
    // [R][Wt][32] staging box (swizzled 16-byte chunks, conflict-free) -> ONE
    // bulk tensor store per 32-column chunk (TMA clips image/tensor edges;
    // reduce-add implements accumulate in place). Double-buffered staging.
    if (warp < 4) {
      pdl_wait();  // Y may still be read by the preceding kernel
      const uint32_t q = warp;
      const int m = static_cast<int>(q * 32 + lane);
      const int ry = m / p.Wv, cx = m - ry * p.Wv;
      const bool mine = ry < p.R && cx < p.Wt;
      const int line = ry * p.Wt + cx;
      const int line_bytes = p.out_f16 ? 64 : 128;
      uint32_t acc = 0, acc_phase = 0, chunk = 0;
      // Bias fetched before the accumulator wait (one column per lane, then
      // shuffled), the residual of the next 32 columns in flight during the
      // current chunk: loads issued next to their use stall the chunk chain.
      const bool epi_on = p.bias || p.relu || p.residual;
      for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x) {
        int n, th, tw, g, nt;
        decompose(tile, n, th, tw, g, nt);
        const int64_t col_tile = static_cast<int64_t>(g) * p.cog + nt * BN;
        const int valid_tile = p.cog - nt * BN;
        // bias of the next 32 columns, one column per lane (prefetched a chunk ahead)
        float bnext = (p.bias && static_cast<int>(lane) < valid_tile) ? __ldg(p.bias + col_tile + lane) : 0.0f;
        const uint16_t* res_row = nullptr;
        if (p.residual && mine) {
          const int oy = th * p.R + ry, ox = tw * p.Wt + cx;
          if (oy < p.oh && ox < p.ow)
            res_row = p.residual + ((static_cast<int64_t>(n) * p.oh + oy) * p.ow + ox) * p.co + col_tile;
        }
        uint4 rp[4];
        auto fetch_res = [&](int c) {
          if (res_row && valid_tile - c >= 32 && (reinterpret_cast<uintptr_t>(res_row + c) & 15) == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) rp[i] = __ldg(reinterpret_cast<const uint4*>(res_row + c) + i);
          }
        };
        fetch_res(0);
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (threadIdx.x == 0 && tile == static_cast<int>(blockIdx.x)) trace_event(p.trace, TR_FIRST_TFULL);
        if (trace && threadIdx.x == 0) trace[512 + 2 * (tile / gridDim.x)] = clock64();
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32, ++chunk) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((q * 32u) << 16) + acc * BN + c0, r);
          tmem_ld_wait();
          if (epi_on) {
            float* v = reinterpret_cast<float*>(r);
            const int lim = valid_tile - c0;
            if (p.bias) {
              const float bcur = bnext;
              const int nc = c0 + 32 + static_cast<int>(lane);
              bnext = nc < valid_tile ? __ldg(p.bias + col_tile + nc) : 0.0f;
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] += __shfl_sync(0xffffffffu, bcur, i);
            }
            if (res_row) {
              if (lim >= 32 && (reinterpret_cast<uintptr_t>(res_row + c0) & 15) == 0) {
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
                        __ldg(reinterpret_cast<const unsigned short*>(res_row + c0) + i)));
              }
              fetch_res(c0 + 32);
            }
            epi_act_n<32>(v, p.relu);
          }
          uint8_t* buf = epi + (chunk & 1) * p.stage_bytes;
          named_bar_sync(1, 128);  // buffer (chunk & 1) no longer read by an older store
          if (mine) {
            uint8_t* dst = buf + line * line_bytes;
            if (p.out_f16) {
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
                *reinterpret_cast<uint4*>(dst + ((c ^ ((line >> 1) & 3)) << 4)) = u;  // SW64
              }
            } else {
#pragma unroll
              for (int c = 0; c < 8; ++c)
                *reinterpret_cast<uint4*>(dst + ((c ^ (line & 7)) << 4)) =
                    make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);  // SW128
            }
          }
          fence_proxy_async_smem();
          named_bar_sync(2, 128);
          if (threadIdx.x == 0) {
            const int col = g * p.cog + nt * BN + c0;
            if (p.store_mode == 2)
              tma_reduce_add_4d(&p.tmY, buf, col, tw * p.Wt, th * p.R, n);
            else
              tma_store_4d(&p.tmY, buf, col, tw * p.Wt, th * p.R, n);
            tma_store_commit();
            tma_store_wait_read<1>();
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        if (trace && threadIdx.x == 0) trace[513 + 2 * (tile / gridDim.x)] = clock64();
        if (++acc == static_cast<uint32_t>(Cfg::kNacc)) {
          acc = 0;
          acc_phase ^= 1;
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
  } else {
    // ------------------------------------------------------------ epilogue (warps 0-7)
    // Warp e owns TMEM lanes 32*(e%4) + 16*(e/4) .. +15 (16 tile rows) and reads
    // them with tcgen05.ld.16x256b: four consecutive threads hold 8 consecutive
    // fp32 columns of one row, so every store instruction writes whole 32-byte
    // sectors (8 rows x 32 B) straight from registers — no smem staging (the
    // kernel is shared-memory-bandwidth bound: MMA operand reads already use it).
    const uint32_t q = warp & 3, hh = warp >> 2;
    const uint32_t lane0 = q * 32 + hh * 16;
    const int r_lo = static_cast<int>(lane0 + lane / 4), r_hi = r_lo + 8;
    const int cq = 2 * static_cast<int>(lane % 4);
    pdl_wait();
    uint32_t local = 0, acc = 0, acc_phase = 0;
    for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x, ++local) {
      int n, th, tw, g, nt;
      decompose(tile, n, th, tw, g, nt);
      auto row_offset = [&](int m) -> int64_t {
        const int ry = m / p.Wv, cx = m - ry * p.Wv;
        if (ry >= p.R || cx >= p.Wt) return -1;
        const int oy = th * p.R + ry, ox = tw * p.Wt + cx;
        if (oy >= p.oh || ox >= p.ow) return -1;
        return ((static_cast<int64_t>(n) * p.oh + oy) * p.ow + ox) * p.co + g * p.cog + nt * BN;
      };
      const int64_t off_lo = row_offset(r_lo), off_hi = row_offset(r_hi);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (trace && threadIdx.x == 0 && local < 64) trace[512 + 2 * local] = clock64();
      const int ncol0 = nt * BN;
      constexpr int kCols = BN < 32 ? BN : 32;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += kCols) {
        uint32_t r[16];
        const uint32_t taddr = tmem_base + (lane0 << 16) + acc * BN + c0;
        if constexpr (kCols == 32) tmem_ld_16x256b_x4(taddr, r);
        else tmem_ld_16x256b_x2(taddr, r);
        tmem_ld_wait();
        const int valid = p.cog - (ncol0 + c0);
        if (valid <= 0) continue;
#pragma unroll
        for (int j = 0; j < kCols / 8; ++j) {
          const int col = 8 * j + cq;
          if (col >= valid) continue;
          const bool pair = col + 1 < valid;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t ro = h ? off_hi : off_lo;
            if (ro < 0) continue;
            const int64_t off = ro + c0 + col;
            float v0 = __uint_as_float(r[4 * j + 2 * h]), v1 = __uint_as_float(r[4 * j + 2 * h + 1]);
            if (p.accumulate) {
              if (pair) {
                const float2 t = *reinterpret_cast<const float2*>(p.Yin + off);
                v0 = t.x + v0;
                v1 = t.y + v1;
              } else {
                v0 = p.Yin[off] + v0;
              }
            }
            if (p.bias || p.relu || p.residual) {
              const int64_t colb = g * p.cog + ncol0 + c0 + col;
              float vv[2] = {v0, v1};
              epi_run<2>(vv, p.bias, colb, pair ? 2 : 1, p.residual ? p.residual + off : nullptr, p.relu);
              v0 = vv[0];
              v1 = vv[1];
            }
            if (p.out_f16) {
              __half* y = reinterpret_cast<__half*>(p.Y) + off;
              if (pair) *reinterpret_cast<__half2*>(y) = __floats2half2_rn(v0, v1);
              else y[0] = __float2half_rn(v0);
            } else {
              float* y = reinterpret_cast<float*>(p.Y) + off;
              if (pair) *reinterpret_cast<float2*>(y) = make_float2(v0, v1);
              else y[0] = v0;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (trace && threadIdx.x == 0 && local < 64) trace[512 + 2 * local + 1] = clock64();
      if (++acc == static_cast<uint32_t>(Cfg::kNacc)) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc(tmem_base, Cfg::kTmemCols);
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
