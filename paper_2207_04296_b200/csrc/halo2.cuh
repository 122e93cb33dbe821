// halo2.cuh — the halo-tile stride-1 convolution (halo.cuh) on CTA pairs:
// tcgen05.mma.cta_group::2, M = 256 per MMA (two 128-pixel tiles, one per SM of
// a TPC), N = 64, weights split by output column across the pair.
//
// Why: the N = 64 headline conv is bound by the SM's shared-memory read port
// inside the MMA (A 4 KB + B 2 KB per 128x64x16 MMA, measured 48 instead of 32
// cycles, tools/mma_rate.cu; ~2450 cycles per tile, tools/trace_igemm.py). With
// a CTA pair each SM feeds its own A but only half of B (32 of the 64 weight
// columns): 5 instead of 6 KB per MMA, and each CTA keeps half the resident
// weights (37 instead of 74 KB of shared memory).
//
// Pipeline (everything else as in halo.cuh):
//   * cluster of 2; rank 0 (leader) issues every MMA for both CTAs; CTA r of
//     pair iteration j computes tile 2*(cluster + j*clusters) + r;
//   * each CTA's producer TMA-loads its own slab (and its half of the weights)
//     with the .cta_group::2 form, completing on the LEADER's full / weight
//     barriers (shared::cluster address with the peer bit cleared); the leader's
//     producer posts the expected bytes of both CTAs;
//   * the leader's commits multicast to both CTAs' empty / tfull barriers;
//   * both CTAs' epilogue warps drain their own TMEM lanes and arrive on the
//     leader's tempty barrier (remote arrive for rank 1);
//   * TMEM is allocated and freed with cta_group::2 in both CTAs; cluster
//     barriers fence initialisation and teardown.
// Shapes: 3x3 (any KH x KW), dilation, padding, 64 output channels in one group,
// TMA-store epilogue (store modes 1 / 2), rectangular tiles.
#pragma once

#include "halo.cuh"

namespace tb {

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of the leader CTA's copy of a barrier (peer bit cleared)
__device__ __forceinline__ uint32_t leader_addr(const void* p) { return smem_u32(p) & 0xFEFFFFFFu; }

__device__ __forceinline__ void tma_load_4d_pair(void* dst, const CUtensorMap* m, uint32_t leader_bar, int c0,
                                                 int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint32_t leader_bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrives on `bar` (same offset) in both CTAs of the pair once the issued MMAs complete.
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

constexpr int kPairBN = 64;                      // N of one pair MMA (output channels)
constexpr int kPairBHalf = 32;                   // weight columns resident per CTA
constexpr uint32_t kPairIdesc = idesc_f16_f32(256, kPairBN, 0, 1);
constexpr int kPairNacc = 4;
constexpr int kPairTmemCols = 256;

inline size_t halo2_smem_bytes(int stages, int slab_rows, int b_rows, int stage_bytes) {
  return 1024 + static_cast<size_t>(stages) * slab_rows * 128 + static_cast<size_t>(b_rows) * kPairBHalf * 2 +
         2 * static_cast<size_t>(stage_bytes) + 256;
}

__global__ void __launch_bounds__(kHaloThreads, 1) conv_halo2_kernel(const __grid_constant__ HaloParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int S = p.stages;
  const uint32_t slab_bytes = static_cast<uint32_t>(p.slab_rows) * 128;
  uint8_t* sA0 = smem;
  uint8_t* sB = smem + static_cast<size_t>(S) * slab_bytes;  // [b_rows][32 cols] SW64
  uint8_t* epi = sB + static_cast<size_t>(p.b_rows) * kPairBHalf * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + 2 * p.stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + kPairNacc;
  uint64_t* bfull = tempty + kPairNacc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster = static_cast<int>(blockIdx.x) / 2, nclusters = static_cast<int>(gridDim.x) / 2;
  const int total_pairs = (p.total_tiles + 1) / 2;
  const int my_pairs = cluster < total_pairs ? (total_pairs - 1 - cluster) / nclusters + 1 : 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);   // leader: its producer posts both CTAs' bytes
      mbar_init(&empty[i], 1);  // one multicast commit per phase
    }
    for (int i = 0; i < kPairNacc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);  // leader: 4 epilogue warps x 2 CTAs
    }
    mbar_init(bfull, 1);
    fence_barrier_init();
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kPairTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peers' barriers initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[1023] = clock64();
  uint64_t t_start = 0;
  if (p.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

  auto decompose = [&](int tile, int& n, int& th, int& tw) {
    int r = tile;
    tw = r % p.tiles_w;
    r /= p.tiles_w;
    th = r % p.tiles_h;
    n = r / p.tiles_h;
  };
  auto tile_of = [&](int j, bool& valid) {
    const int t = 2 * (cluster + j * nclusters) + static_cast<int>(rank);
    valid = t < p.total_tiles;
    return valid ? t : p.total_tiles - 1;  // an odd tail: load a real slab, skip its store
  };

  if (warp == 8) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (elect_one()) {
      pdl_wait();  // X / W may be produced by the preceding kernel
      const uint32_t slab_tx = static_cast<uint32_t>(p.HR) * p.Wv * 128;
      if (my_pairs > 0) {
        // this CTA's half of the weights: columns [32 * rank, 32 * rank + 32), all rows
        if (leader) mbar_arrive_expect_tx(bfull, 2u * static_cast<uint32_t>(p.b_rows) * kPairBHalf * 2);
        for (int r = 0; r < p.b_rows; r += p.b_box_rows)
          tma_load_2d_pair(sB + static_cast<size_t>(r) * kPairBHalf * 2, &p.tmW, leader_addr(bfull),
                           static_cast<int>(rank) * kPairBHalf, r);
      }
      uint32_t slot = 0, phase = 0;
      for (int j = 0; j < my_pairs; ++j) {
        bool valid;
        int n, th, tw;
        decompose(tile_of(j, valid), n, th, tw);
        const int y0 = th * p.R - p.pad_h, x0 = tw * p.Wt - p.pad_w;
        for (int cb = 0; cb < p.cblocks; ++cb) {
          mbar_wait(&empty[slot], phase ^ 1);
          if (p.trace && blockIdx.x == 0 && j * p.cblocks + cb < 128) p.trace[2 * (j * p.cblocks + cb)] = clock64();
          if (leader) mbar_arrive_expect_tx(&full[slot], 2 * slab_tx);
          tma_load_4d_pair(sA0 + slot * slab_bytes, &p.tmX, leader_addr(&full[slot]), cb * 64, x0, y0, n);
          if (++slot == static_cast<uint32_t>(S)) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader && my_pairs > 0) {
      const uint64_t a0 = smem_desc(smem_u32(sA0), 16, 1024, 2);
      // B: [rows][32 cols] MN-major SW64 (64-byte rows, 8-row groups of 512 B)
      const uint64_t b0 = smem_desc(smem_u32(sB), p.b_rows * kPairBHalf * 2, 512, 4);
      const uint32_t slab16 = slab_bytes >> 4;
      const int wv_dil = p.Wv * p.dil * 8;
      const int dil8 = p.dil * 8;
      const int cig_b = (p.cig * kPairBHalf * 2) >> 4;   // one tap's weight rows
      constexpr uint32_t kBk16 = (16 * kPairBHalf * 2) >> 4;
      const int taps = p.kh * p.kw;
      mbar_wait(bfull, 0);
      tc_fence_after();
      const int nstage = my_pairs * p.cblocks;
      unsigned long long* trace = (blockIdx.x == 0) ? p.trace : nullptr;
      uint32_t slot = 0, phase = 0, acc = 0, acc_phase = 0;
      // As in halo.cuh: the next stage's barriers are waited on after all but the
      // last tap of this stage is issued, so the tensor pipe does not drain.
      auto wait_stage = [&](int i, uint32_t sl, uint32_t ph, uint32_t ac, uint32_t acph) {
        if (i % p.cblocks == 0) mbar_wait(&tempty[ac], acph ^ 1);
        mbar_wait(&full[sl], ph);
        tc_fence_after();
      };
      if (nstage > 0) wait_stage(0, 0, 0, 0, 0);
      for (int i = 0; i < nstage; ++i) {
        const int cb = i % p.cblocks;
        const bool last_cb = cb == p.cblocks - 1;
        uint32_t nslot = slot + 1, nphase = phase, nacc = acc, nacc_phase = acc_phase;
        if (nslot == static_cast<uint32_t>(S)) { nslot = 0; nphase ^= 1; }
        if (last_cb && ++nacc == static_cast<uint32_t>(kPairNacc)) { nacc = 0; nacc_phase ^= 1; }
        if (trace && lane == 0 && i < 128) trace[256 + 2 * i] = clock64();
        const uint32_t tmem_d = tmem_base + acc * kPairBN;
        const uint64_t a_slab = a0 + slot * slab16;
        const uint64_t b_cb = b0 + ((static_cast<uint32_t>(cb * 64) * kPairBHalf * 2) >> 4);
        auto issue_tap = [&](int t) {
          const int ty = t / p.kw, tx = t - ty * p.kw;
          const uint64_t a = a_slab + static_cast<uint32_t>(ty * wv_dil + tx * dil8);
          const uint64_t b = b_cb + static_cast<uint32_t>(t * cig_b);
#pragma unroll
          for (int k = 0; k < 4; ++k) umma_f16_pair(tmem_d, a + 2u * k, b + k * kBk16, kPairIdesc, (cb | t | k) != 0);
        };
        const bool issuer = elect_one();
        if (issuer)
          for (int t = 0; t < taps - 1; ++t) issue_tap(t);
        __syncwarp();
        if (i + 1 < nstage) wait_stage(i + 1, nslot, nphase, nacc, nacc_phase);
        if (issuer) {
          issue_tap(taps - 1);
          umma_commit_pair(&empty[slot]);
          if (last_cb) umma_commit_pair(&tfull[acc]);
        }
        __syncwarp();
        if (trace && lane == 0 && i < 128) trace[256 + 2 * i + 1] = clock64();
        slot = nslot; phase = nphase; acc = nacc; acc_phase = nacc_phase;
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ epilogue, TMA store (both CTAs)
    pdl_wait();  // Y may still be read by the preceding kernel
    const uint32_t q = warp;
    const int m = static_cast<int>(q * 32 + lane);
    const int ry = m / p.Wv, cx = m - ry * p.Wv;
    const bool mine = ry < p.R && cx < p.Wt;
    const int line = ry * p.Wt + cx;
    const int line_bytes = p.out_f16 ? 64 : 128;
    const bool epi_on = p.bias || p.relu || p.residual;
    uint32_t acc = 0, acc_phase = 0, chunk = 0;
    for (int j = 0; j < my_pairs; ++j) {
      bool valid;
      int n, th, tw;
      decompose(tile_of(j, valid), n, th, tw);
      float bnext = (p.bias && static_cast<int>(lane) < p.cog) ? __ldg(p.bias + lane) : 0.0f;
      const uint16_t* res_row = nullptr;
      if (p.residual && mine && valid) {
        const int oy = th * p.R + ry, ox = tw * p.Wt + cx;
        if (oy < p.oh && ox < p.ow) res_row = p.residual + ((static_cast<int64_t>(n) * p.oh + oy) * p.ow + ox) * p.co;
      }
      uint4 rp[4];
      auto fetch_res = [&](int c) {
        if (res_row && (reinterpret_cast<uintptr_t>(res_row + c) & 15) == 0) {
#pragma unroll
          for (int i = 0; i < 4; ++i) rp[i] = __ldg(reinterpret_cast<const uint4*>(res_row + c) + i);
        }
      };
      fetch_res(0);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < kPairBN; c0 += 32, ++chunk) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((q * 32u) << 16) + acc * kPairBN + c0, r);
        tmem_ld_wait();
        if (c0 + 32 >= kPairBN) {  // accumulator fully read: release it to the leader's MMA
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive(&tempty[acc]);
            else mbar_arrive_leader(&tempty[acc]);
          }
        }
        if (epi_on) {
          float* v = reinterpret_cast<float*>(r);
          if (p.bias) {
            const float bcur = bnext;
            const int nc = c0 + 32 + static_cast<int>(lane);
            bnext = nc < p.cog ? __ldg(p.bias + nc) : 0.0f;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += __shfl_sync(0xffffffffu, bcur, i);
          }
          if (res_row) {
            if ((reinterpret_cast<uintptr_t>(res_row + c0) & 15) == 0) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const __half2* hv = reinterpret_cast<const __half2*>(&rp[i]);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  const float2 f = __half22float2(hv[jj]);
                  v[8 * i + 2 * jj] += f.x;
                  v[8 * i + 2 * jj + 1] += f.y;
                }
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                v[i] += __half2float(__ushort_as_half(__ldg(reinterpret_cast<const unsigned short*>(res_row + c0) + i)));
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
        if (threadIdx.x == 0 && valid) {
          if (p.store_mode == 2)
            tma_reduce_add_4d(&p.tmY, buf, c0, tw * p.Wt, th * p.R, n);
          else
            tma_store_4d(&p.tmY, buf, c0, tw * p.Wt, th * p.R, n);
          tma_store_commit();
        }
        if (threadIdx.x == 0) tma_store_wait_read<1>();
      }
      if (++acc == static_cast<uint32_t>(kPairNacc)) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (threadIdx.x == 0) tma_store_wait_read<0>();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the leader's MMAs into this CTA's TMEM are done before it is freed
  tc_fence_after();
  if (warp == 9)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kPairTmemCols)
                 : "memory");
  if (p.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
    uint64_t t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    p.trace[2048 + 4 * blockIdx.x] = t_start;
    p.trace[2048 + 4 * blockIdx.x + 1] = t_end;
    p.trace[2048 + 4 * blockIdx.x + 3] = my_pairs;
  }
}

}  // namespace tb
