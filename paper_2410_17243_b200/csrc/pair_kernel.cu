// The fused Inf-CL tile kernel for sm_100a: one persistent CTA pair per two SMs.
//
// A pair owns a block of 128 stationary rows (64 per SM, resident in smem) and streams 256-column tiles of
// the other side through a TMA ring.  Per tile:
//   S GEMM   : S (128 x 256) = A_R * B_C^T, K = d, tcgen05.mma.cta_group::2 M=128 N=256 ("2x2" TMEM
//              layout: per SM 64 rows x 256 cols held as 128 lanes x 128 cols).            [Eq.3, Alg.2 l.8]
//   forward  : epilogue folds the tile into running row (m, sigma) states in registers (Eq.5 + Eq.4,
//              Alg.2 l.9-12) and computes exact column (max, sum) partials with warp-shuffle transposed
//              reductions, merged into a per-CTA column slot (symmetric text->image direction).
//   backward : epilogue recomputes G_ij = 2^{y-r2_i} + 2^{y-c2_j} (Alg.4 l.11, Eq.7-8), rounds to bf16 and
//              stores it to smem; then dA^T (d x 128) += B_C^T * G^T with tcgen05.mma.cta_group::2 M=256
//              (d split across the pair: 128 d-rows per SM), N=128, K=256, B_C read MN-major from the same
//              TMA tiles layout.  The dA accumulator stays in TMEM across the whole row block (Alg.4
//              l.12 "dI += ..."), and is drained with red.add at the end of the row block.
// Warp roles (320 threads): warps 0-7 epilogue (TMEM lane quarter = warp % 4, column slice = warp / 4), warp 8 TMA
// producer, warp 9 TMEM alloc + MMA issuer (leader CTA).  The issuers get the highest warp ids because the warp
// arbiter favours higher ids: they must not lose issue slots to the epilogue warps sharing their sub-partition.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <utility>
#include <vector>

#include "host_utils.h"
#include "kernels.h"
#include "pair_common.cuh"
#include "ptx.cuh"

namespace infcl {

// ---- optional per-launch event timing (infcl_profile_*)
struct ProfState {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[3];  // 0 fwd kernel, 1 bwd kernel, 2 ring block send
};
static ProfState& prof() {
  static ProfState p;
  return p;
}
static void prof_clear() {
  for (auto& v : prof().ev)
    for (auto& e : v) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  for (auto& v : prof().ev) v.clear();
}

// Consumer CTA pair of the fused backward (GC): for every wave w of gc_pp row blocks and each of its units (column
// tile ct, d-chunk part) u = c, c + P_c, ... (c = pair - gc_pp, P_c = npairs - gc_pp; a unit's consumer is the same in
// every wave, so each dB element receives its per-wave partials from one thread in wave order: deterministic),
// accumulate
//   dB (256 columns j x 256-d chunks) += G_w,t^T (j x 128 rows i) * A_w,t (128 rows i x d)   over the wave's tiles t
// with tcgen05.mma.cta_group::2 M=256 (128 columns j per SM) N=256 K=16, both operands MN-major: G tiles from the
// global ring (tmG, boxes of 64 rows x 64 columns), A rows (tmI, boxes of 128 rows x 64 features), one ring of 32-KB
// stages (per tile: one G stage, then one stage per d chunk).  TMEM lane = column j, TMEM column = feature d, so the
// drain (once per unit and wave, scaled by s g / 2b) adds 4 consecutive features per red.global.add.v4.f32.  This is
// Alg.4's dT~ update with the G tiles handed over through memory instead of a read-modify-write of dT
// per tile.
template <bool DBG>
__device__ __forceinline__ void gc_consumer(const CUtensorMap* tmG, const CUtensorMap* tmI, const CUtensorMap* tmDT,
                                            const KParams& p,
                                            uint8_t* smem, uint64_t* full, uint64_t* empty, uint64_t* dafull,
                                            uint64_t* dafree, uint32_t tbase, int warp, int lane, uint32_t cta,
                                            int pair) {
  const int PP = p.gc_pp, PC = p.npairs - p.gc_pp, c = pair - p.gc_pp;
  const int nW = (p.n_rb + PP - 1) / PP;
  // units u = ct * nparts + part: part 0 = d chunks [0, 2), part 1 = [2, NDC) (d > 512: the accumulator of a
  // whole 768-wide column tile exceeds TMEM); unit u belongs to consumer u mod PC in every wave
  const int nparts = p.NDC > 2 ? 2 : 1, nunits = p.n_ct * nparts;
  // items k = wave * nunits + unit go round-robin over the consumers (consumer c: k = c, c + P_c, ...)
  const long long nitems = (long long)nW * nunits;
  const int nsc = p.n_stages_c;
  if (warp == kWarpTMA) {
    if (lane == 0) {
      WaitClock<DBG> wc(p.dbg, true);
      const uint64_t polG = (p.gc_hint & 1) ? policy_evict_first() : policy_evict_normal();
      const uint64_t polA = (p.gc_hint & 4) ? policy_evict_last() : policy_evict_normal();
      int stage = 0;
      uint32_t ph = 0;
      auto acquire = [&]() -> uint8_t* {
        wc.wait(&empty[stage], ph ^ 1u, 1);
        if (cta == 0) mbar_arrive_expect_tx(&full[stage], 2 * 32768);
        return smem + stage * 32768;
      };
      auto advance = [&]() {
        if (++stage == nsc) {
          stage = 0;
          ph ^= 1;
        }
      };
      for (long long kk = c; kk < nitems; kk += PC) {
        const int w = (int)(kk / nunits), un = (int)(kk % nunits);
        const int nt = min(PP, p.n_rb - w * PP);
        {
          const int ct = un / nparts, tc0 = (un % nparts) * 2, tc1 = min(p.NDC, tc0 + 2);
          const long long g = (long long)w * p.n_ct + ct;
          const int slot_row = (int)((g % p.gc_ring) * PP) * kRowsPerPair;
          // the unit's dB rows (its 128 columns j of this CTA, whole rows) are pulled into L2 a few tiles before
          // the drain: a wave-old dB tile has left L2, and the drain's reductions would wait on HBM
          const int t_pf = max(0, nt - 12);
          for (int t = 0; t < nt; ++t) {
            if (t == t_pf) {
              const int j0 = ct * kColsPerTile + (int)cta * 128, nj = min(128, p.ncols - j0);
              if (nj > 0) {
                const char* base = reinterpret_cast<const char*>(p.dB + (long long)j0 * p.ld_dB);
                const long long bytes = (long long)nj * p.ld_dB * 4;
                for (long long o = 0; o < bytes; o += 65536)
                  prefetch_l2_bulk(base + o, (uint32_t)std::min<long long>(65536, bytes - o));
              }
            }
            // tile t of step g is in the ring once both CTAs of producer pair t published it
            const unsigned long long t_sp = DBG ? clock64() : 0ull;
            spin_geq(p.g_ready + g * PP + t, 2u, 14);
            if (DBG) wc.acc[0] += clock64() - t_sp;
            fence_proxy_async_global();
            uint8_t* gd = acquire();  // G stage: boxes (ib, jb) at (2 ib + jb) * 8 KB
#pragma unroll
            for (int ib = 0; ib < 2; ++ib)
#pragma unroll
              for (int jb = 0; jb < 2; ++jb)
                tma_load_2d_pair_hint(gd + (2 * ib + jb) * kBox, tmG, &full[stage], ((int)cta * 2 + jb) * 64,
                                      slot_row + t * kRowsPerPair + ib * 64, polG);
            advance();
            const int r0 = (w * PP + t) * kRowsPerPair;
            for (int tc = tc0; tc < tc1; ++tc) {
              uint8_t* dst = acquire();  // this CTA's 128 features of chunk tc x the tile's 128 rows
              const int d0 = tc * 256 + (int)cta * 128;
              tma_load_2d_pair_hint(dst, tmI, &full[stage], d0, r0, polA);
              tma_load_2d_pair_hint(dst + kBoxB, tmI, &full[stage], d0 + 64, r0, polA);
              advance();
            }
          }
        }
      }
      wc.flush(5);
    }
  } else if (warp == kWarpMMA) {
    if (cta == 0) {
      WaitClock<DBG> wc(p.dbg, lane == 0);
      const unsigned long long t_loop = DBG ? clock64() : 0ull;
      const uint32_t idT = idesc_bf16(256, 256, 1, 1);
      int stage = 0;
      uint32_t ph = 0, dph = 0;
      auto advance = [&]() {
        if (++stage == nsc) {
          stage = 0;
          ph ^= 1;
        }
      };
      for (long long kk = c; kk < nitems; kk += PC) {
        const int w = (int)(kk / nunits), un = (int)(kk % nunits);
        const int nt = min(PP, p.n_rb - w * PP);
        {
          const int ct = un / nparts, tc0 = (un % nparts) * 2, tc1 = min(p.NDC, tc0 + 2);
          const long long g = (long long)w * p.n_ct + ct;
          wc.wait(dafree, dph ^ 1u, 3, true);
          dph ^= 1;
          tc_fence_after();
          for (int t = 0; t < nt; ++t) {
            const int gs = stage;
            wc.wait(&full[gs], ph, 4);
            tc_fence_after();
            // the tile (both CTAs' halves) is in smem: with one reader per tile (d <= 512) its 64 KB of ring lines
            // are dead -- drop them from L2 without a write-back (hint bit 16: keep them); after the step's last
            // tile the slot may be refilled
            if (nparts == 1 && !(p.gc_hint & 16)) {
              const uint16_t* tl = p.g_ring + ((g % p.gc_ring) * PP + t) * (long long)(kRowsPerPair * kColsPerTile);
#pragma unroll
              for (int i = 0; i < 16; ++i) discard_l2_line(tl + (i * 32 + lane) * 64);
            }
            if (t == nt - 1 && lane == 0) red_release_gpu_add(p.g_consumed + g, 1u);
            __syncwarp();
            const uint32_t a_lo = (uint32_t)smem_desc_sw128(smem_u32(smem + gs * 32768), kBox, 1024);  // LBO: jb
            advance();
            for (int tc = tc0; tc < tc1; ++tc) {
              wc.wait(&full[stage], ph, 5);
              tc_fence_after();
              const uint32_t b_lo = (uint32_t)smem_desc_sw128(smem_u32(smem + stage * 32768), kBoxB, 1024);
              umma_stage_dT_pair(tbase + (tc - tc0) * 256, a_lo, b_lo, idT, t != 0 ? 1u : 0u);
              umma_commit_pair_mc_warp(&empty[stage], 0x3);
              advance();
            }
            umma_commit_pair_mc_warp(&empty[gs], 0x3);
          }
          umma_commit_pair_mc_warp(dafull, 0x3);
        }
      }
      if (DBG) wc.acc[0] += clock64() - t_loop;
      wc.flush(6);
    }
  } else if (warp < 8) {
    // drain: warp (q, u) holds columns j = ct*256 + cta*128 + 32q + lane, features 128u .. 128u + 127 of each chunk
    const int q = warp & 3, u = warp >> 2;
    const float coef = p.coef_base * __ldg(p.grad);
    WaitClock<DBG> wc(p.dbg, lane == 0);
    const uint32_t stg_off = (uint32_t)nsc * 32768 + warp * 4096;  // this warp's staging box (after the ring)
    const uint32_t stg = smem_u32(smem) + stg_off;
    uint32_t daph = 0;
    for (long long kk = c; kk < nitems; kk += PC) {
      const int w = (int)(kk / nunits), un = (int)(kk % nunits);
      {
        const int ct = un / nparts, tc0 = (un % nparts) * 2, tc1 = min(p.NDC, tc0 + 2);
        wc.wait(dafull, daph, 10, true);
        daph ^= 1;
        const unsigned long long t_dr = DBG ? clock64() : 0ull;
        tc_fence_after();
        // each 32 x 32 block (columns j of this warp's lanes, 32 features) goes through the warp's 4-KB staging
        // box (128-B swizzle: conflict-free v4 stores) and a TMA reduce-add into dB (the tensor map clips the
        // ragged columns j >= ncols and features >= d_out)
        const int j0 = ct * kColsPerTile + (int)cta * 128 + q * 32;
        // waves reach each dB element in wave order (bitwise reproducible dB): this unit's previous wave, drained
        // by whichever consumer had it, has completed all 16 warps' reductions (long since, as a rule)
        if (w > 0) {
          if (lane == 0) {
            spin_geq(p.g_unit_done + un, 16u * (uint32_t)w, 17);
            fence_proxy_async_global();
          }
          __syncwarp();
        }
        for (int tc = tc0; tc < tc1; ++tc) {
          for (int cc = 0; cc < 4; ++cc) {
            const int col0 = u * 128 + cc * 32;
            float y[32];
            tmem_ld32(tbase + ((uint32_t)(q * 32) << 16) + (tc - tc0) * 256 + col0, y);
            tmem_ld_wait();
            if (lane == 0) bulk_wait_read<0>();  // the previous block has left the staging box
            __syncwarp();
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4)
              st_shared_v4f(stg + lane * 128 + ((c4 ^ (lane & 7)) << 4), coef * y[4 * c4], coef * y[4 * c4 + 1],
                            coef * y[4 * c4 + 2], coef * y[4 * c4 + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && !(DBG && (p.gc_hint & 8))) {  // hint bit 8 (debug builds): no drain (invalid dB)
              tma_reduce_add_2d(tmDT, smem + stg_off, tc * 256 + col0, j0);
              bulk_commit();
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cluster(dafree, 0);
          bulk_wait<0>();  // this warp's reductions of the unit are done: the unit's next wave may follow
          red_release_gpu_add(p.g_unit_done + un, 1u);
        }
        if (DBG) wc.acc[6] += clock64() - t_dr;
      }
    }
    if (lane == 0) bulk_wait<0>();  // every reduction of this warp has landed before the kernel ends
    wc.flush(7);
  }
}

template <bool BWD, bool DBG, bool GC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GC ? kThreadsGC : kThreads, 1)
    pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmI,
                const __grid_constant__ CUtensorMap tmGs, const __grid_constant__ CUtensorMap tmDT,
                const __grid_constant__ KParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];  // SW128 operands need 1024-B alignment
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u)) __trap();  // fail loudly, never silently misalign
  uint8_t* sA = smem;
  uint8_t* sG = sA + p.KB * kBox;
  uint8_t* sStage = sG + (BWD ? 4 * kBox : 0);

  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  // S buffers in TMEM: forward 4 x 128 columns (MMA up to 3 tiles ahead); backward one 128-column buffer in front
  // of the dA accumulator (a second one where TMEM allows, d <= 512, measured 1-3 % slower: DESIGN.md perf log)
  constexpr int kNB = BWD ? 1 : 4;
  __shared__ __align__(8) uint64_t afull, afree, sfull[kNB], sfree[kNB], gready, gfree, dafull, dafree;
  __shared__ uint32_t tmem_base;
  // fused backward producers: steps g <= gc_free_upto have a free ring slot; epilogue warps that wrote their tile rows
  __shared__ long long gc_free_upto;
  __shared__ uint32_t gc_written;
  __shared__ __align__(16) float2 xch[2][4][2][64];  // forward column partials of a group's 2 warps (x tile parity)
  __shared__ float2 rowx[4][64];                  // forward row partials of the 4 column slices
  __shared__ __align__(16) float cval[8][64];     // backward: each warp's 64 column LSEs (log2)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  // fused backward: pairs >= gc_pp are consumers of the G ring (gc_consumer below)
  const bool consumer = GC && pair >= p.gc_pp;
  const Sched S(p.n_rb, p.n_ct, GC ? p.gc_pp : p.npairs, pair, GC);
  const long long nk = S.n_local();
  constexpr uint32_t kTmemCols = 512;

  if (threadIdx.x == 0) {
    // (GC: the consumer CTAs use n_stages_c ring stages of the same arrays)
    for (int s = 0; s < (consumer ? p.n_stages_c : p.n_stages); ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&afull, 1);
    mbar_init(&afree, 1);
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&sfull[b], 1);
      mbar_init(&sfree[b], 16);  // one arrival per epilogue warp of both CTAs
    }
    gc_free_upto = GC ? (long long)p.gc_ring - 1 : 0;
    gc_written = 0;
    mbar_init(&gready, 16);
    mbar_init(&gfree, 1);
    mbar_init(&dafull, 1);
    mbar_init(&dafree, 16);

    fence_mbar_init();
  }
  if (warp == kWarpTMA && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (GC && consumer) {
      tma_prefetch_desc(&tmG);
      tma_prefetch_desc(&tmI);
      tma_prefetch_desc(&tmDT);
    }
    if (GC && !consumer) tma_prefetch_desc(&tmGs);
  }
  if (warp == kWarpMMA) tmem_alloc<2>(&tmem_base, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_base;

  const unsigned long long t_start = DBG ? clock64() : 0ull;
  if (GC && consumer) {
    gc_consumer<DBG>(&tmG, &tmI, &tmDT, p, smem, full, empty, &dafull, &dafree, tbase, warp, lane, cta, pair);
  } else if (GC && warp == kWarpSignal) {
    // ===================================================================== G ring signals (fused backward)
    // one lane keeps gc_free_upto (steps whose ring slot the consumers have read; polled from g_consumed) and
    // publishes each finished tile: once the 8 epilogue warps counted it in gc_written, ready[g] += 1 with
    // gpu-scope release (cumulative over their writes, acquired at CTA scope)
    if (lane == 0) {
      const uint32_t nparts = p.NDC > 2 ? 2u : 1u;
      const long long n_steps = (long long)((p.n_rb + p.gc_pp - 1) / p.gc_pp) * p.n_ct;
      long long fu = (long long)p.gc_ring - 1, k = 0;
      const unsigned long long t0 = clock64();
      unsigned long long t_last = t0;
      while (k < nk) {
        bool moved = false;
        while (fu + 1 < n_steps && ld_acquire_gpu(p.g_consumed + (fu + 1 - p.gc_ring)) >= nparts) {
          ++fu;
          moved = true;
        }
        if (moved) st_volatile_shared(&gc_free_upto, fu);
        const uint32_t wr = ld_acquire_cta_shared(&gc_written);
        while (k < nk && wr >= 8u * (uint32_t)(k + 1)) {
          int rb, ct;
          S.decode(k, rb, ct);
          fence_acq_rel_gpu();
          const int w = rb / p.gc_pp;
          red_release_gpu_add(p.g_ready + ((long long)w * p.n_ct + ct) * p.gc_pp + (rb - w * p.gc_pp), 1u);
          ++k;
          moved = true;
        }
        if (moved) {
          t_last = clock64();
        } else {
          __nanosleep(32);
          if (clock64() - t_last > INFCL_WATCHDOG_CYCLES) watchdog_fire(16, (uint32_t)k);
        }
      }
    }
  } else if (warp == kWarpTMA) {
    // ===================================================================== TMA producer (both CTAs)
    if (lane == 0) {
      WaitClock<DBG> wc(p.dbg, lane == 0);
      int stage = 0;
      uint32_t ph = 0, aph = 0;
      auto load_stage = [&](int c0a, int c1a, int c0b, int c1b) {
        ring_acquire(wc, empty, stage, ph, p.pair_commit);
        if (DBG && p.notma) {
          if (cta == 0) mbar_arrive(&full[stage]);
        } else {
          if (cta == 0) mbar_arrive_expect_tx(&full[stage], 2 * p.stage_bytes);
          uint8_t* dst = sStage + stage * p.stage_bytes;
          tma_load_2d_pair(dst, &tmB, &full[stage], c0a, c1a);
          if (BWD || p.sbox == 2) tma_load_2d_pair(dst + kBoxB, &tmB, &full[stage], c0b, c1b);
        }
        if (++stage == p.n_stages) {
          stage = 0;
          ph ^= 1;
        }
      };
      // S stage kc: this CTA's 128 columns j, d-blocks sbox*kc (and sbox*kc + 1) (K-major operand, K = d)
      auto load_S = [&](int ct) {
        const int j0 = ct * kColsPerTile + (int)cta * 128;
        const int sb = BWD ? 2 : p.sbox;
        for (int kc = 0; kc < p.KC; ++kc) load_stage(kc * sb * 64, j0, kc * sb * 64 + 64, j0);
      };
      // dA stage (tc, jc): 128 columns j of the tile, this CTA's 128 d-rows of chunk tc (MN-major operand, K = j)
      auto load_dA = [&](int ct) {
        for (int tc = 0; tc < p.NDC; ++tc) {
          const int d0 = tc * 256 + (int)cta * 128;
          for (int jc = 0; jc < 2; ++jc) load_stage(d0, ct * kColsPerTile + jc * 128, d0 + 64, ct * kColsPerTile + jc * 128);
        }
      };
      long long it = 0;
      while (it < nk) {
        int rb, ct0;
        S.decode(it, rb, ct0);
        const long long seg_end = S.seg_end(it);
        wc.wait(&afree, aph ^ 1, 2);
        aph ^= 1;
        if (DBG && p.notma) {
          if (cta == 0) mbar_arrive(&afull);
        } else {
          if (cta == 0) mbar_arrive_expect_tx(&afull, 2u * p.KB * kBox);
          for (int kb = 0; kb < p.KB; ++kb)
            tma_load_2d_pair(sA + kb * kBox, &tmA, &afull, kb * 64, rb * kRowsPerPair + (int)cta * 64);
        }
        int prev = -1;
        for (int ct = ct0; it < seg_end; ++it, ++ct) {  // a segment's column tiles are consecutive
          load_S(ct);
          if (BWD && prev >= 0) load_dA(prev);
          prev = ct;
        }
        if (BWD) load_dA(prev);
      }
      wc.flush(0);
    }
  } else if (warp == kWarpMMA) {
    // ===================================================================== MMA issuer (leader CTA)
    // the whole warp runs converged (warp-uniform descriptors); elect.sync inside the asm issues
    if (cta == 0) {
      WaitClock<DBG> wc(p.dbg, lane == 0);
      int stage = 0;
      uint32_t ph = 0, aph = 0, gph = 0, dph = 0;
      uint32_t sfph = 0;  // phase bit of sfree[b] = bit b (a register, not a dynamically indexed array)
      int tile_ctr = 0;
      const uint32_t idS = idesc_bf16(128, 256, 0, 0);
      const uint32_t idD = idesc_bf16(256, 128, 1, 0);
      auto advance = [&]() {
        if (++stage == p.n_stages) {
          stage = 0;
          ph ^= 1;
        }
      };
      auto issue_dA = [&](bool first) {
        if (first) {
          wc.wait(&dafree, dph ^ 1, 3, true);
          dph ^= 1;
        }
        wc.wait(&gready, gph, 4, true);
        gph ^= 1;
        tc_fence_after();
        for (int tc = 0; tc < p.NDC; ++tc) {
          for (int jc = 0; jc < 2; ++jc) {
            wc.wait(&full[stage], ph, 5);
            tc_fence_after();
            // descriptors advance by adding (byte offset >> 4) to the start-address field
            const uint64_t ad0 = smem_desc_sw128(smem_u32(sStage + stage * p.stage_bytes), kBoxB, 1024);  // MN-major B_C^T
            const uint64_t bd0 = smem_desc_sw128(smem_u32(sG + jc * 2 * kBox), 16, 1024);           // K-major G
            const uint32_t dD = tbase + 128 + tc * 128;
            umma_stage_dA_pair<(kBox >> 4)>(dD, (uint32_t)ad0, (uint32_t)bd0, idD, (first && jc == 0) ? 0u : 1u);
            ring_release(empty, stage, p.pair_commit);
            advance();
          }
        }
        umma_commit_pair_mc_warp(&gfree, 0x3);
      };
      const unsigned long long t_loop = DBG ? clock64() : 0ull;
      long long it = 0;
      while (it < nk) {
        const long long seg_end = S.seg_end(it);
        wc.wait(&afull, aph, 6, true);
        aph ^= 1;
        tc_fence_after();
        bool have_prev = false, first_dA = true;
        for (; it < seg_end; ++it) {
          const int buf = BWD ? 0 : (tile_ctr & (kNB - 1));
          wc.wait(&sfree[buf], ((sfph >> buf) & 1u) ^ 1u, 7, true);
          sfph ^= 1u << buf;
          tc_fence_after();
          const uint32_t dS = tbase + buf * 128;
          for (int kc = 0; kc < p.KC; ++kc) {
            wc.wait(&full[stage], ph, 5);
            const unsigned long long t_is = DBG ? clock64() : 0ull;
            tc_fence_after();
            const int sb = BWD ? 2 : p.sbox;
            const uint64_t ad0 = smem_desc_sw128(smem_u32(sA + sb * kc * kBox), 16, 1024);
            const uint64_t bd0 = smem_desc_sw128(smem_u32(sStage + stage * p.stage_bytes), 16, 1024);
            if (sb == 2 && 2 * kc + 1 < p.KB)
              umma_stage_pair<true, (kBox >> 4), (kBoxB >> 4)>(dS, (uint32_t)ad0, (uint32_t)bd0, idS, kc != 0);
            else  // one box per stage, or the half-used last stage of an odd number of 64-d blocks
              umma_stage_pair<false, 0, 0>(dS, (uint32_t)ad0, (uint32_t)bd0, idS, kc != 0);
            ring_release(empty, stage, p.pair_commit);
            if (DBG) wc.acc[11] += clock64() - t_is;
            advance();
          }
          const unsigned long long t_c = DBG ? clock64() : 0ull;
          umma_commit_pair_mc_warp(&sfull[buf], 0x3);
          if (it + 1 == seg_end) umma_commit_pair_mc_warp(&afree, 0x3);
          if (DBG) wc.acc[10] += clock64() - t_c;
          ++tile_ctr;
          if (BWD) {
            if (have_prev) {
              issue_dA(first_dA);
              first_dA = false;
            }
            have_prev = true;
          }
        }
        if (BWD) {
          issue_dA(first_dA);
          umma_commit_pair_mc_warp(&dafull, 0x3);
        }
      }
      if (DBG) wc.acc[0] += clock64() - t_loop;
      wc.flush(1);
    }
  } else {
    // ===================================================================== epilogue (both CTAs)
    // 8 warps: warp w reads TMEM lane quarter q = w % 4 (rows) and column slice u = (w - 2) / 4 of 64 columns.
    // 2x2 layout of the S tile: quarter q -> rows 32*(q&1).., tile columns h*128 + u*64 + [0,64), h = q >> 1.
    const int ep = warp;
    const int q = warp & 3;
    const int u = ep >> 2;
    const int h = q >> 1;
    const int rh = q & 1;
    const int r = rh * 32 + lane;  // row within this CTA's 64
    const int grp = h * 2 + u;     // the 2 warps (rh = 0, 1) that share these 64 columns
    const uint32_t laddr = tbase + ((uint32_t)(q * 32) << 16) + u * 64;
    uint32_t sph = 0, gfph = 0, daph = 0;  // sph: phase bit of sfull[b] = bit b
    WaitClock<DBG> wc(p.dbg, lane == 0);
    int tile_ctr = 0;
    const float k2 = p.k2;
    float coef = 0.f;
    if (BWD) {
      coef = p.coef_base * __ldg(p.grad);
    }
    // backward: this warp's column LSEs for the next tile, prefetched into registers one tile ahead
    // (lane l holds columns 2l, 2l+1 of the warp's 64-column slice) -> no cross-warp barrier per tile
    float2 pc = make_float2(0.f, 0.f);
    auto load_pc_ct = [&](int ctn) {
      const int j = ctn * kColsPerTile + h * 128 + u * 64 + 2 * lane;
      pc.x = j < p.ncols ? __ldg(p.lse_col2 + j) : INFINITY;  // +inf: no column (G masked; excluded from cmin)
      pc.y = j + 1 < p.ncols ? __ldg(p.lse_col2 + j + 1) : INFINITY;
    };
    auto load_pc = [&](long long item) {
      int rbn, ctn;
      S.decode(item, rbn, ctn);
      load_pc_ct(ctn);
    };
    if (BWD && nk > 0) load_pc(0);
    long long it = 0;
    while (it < nk) {
      int rb, ct_first;
      S.decode(it, rb, ct_first);
      const long long seg_end = S.seg_end(it);
      const int ig = rb * kRowsPerPair + (int)cta * 64 + r;
      const bool row_ok = ig < p.nrows;
      // forward (16x256b layout): running (m, sigma) of this thread's 4 rows over its 16-column slice
      float mrow[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, srow[4] = {0.f, 0.f, 0.f, 0.f};
      float r2 = 0.f, rmax = -INFINITY;  // backward: row LSE (log2) and its maximum over the warp's valid rows
      if (BWD) {
        if (row_ok) r2 = __ldg(p.lse_row2 + ig);
        rmax = row_ok ? r2 : -INFINITY;
#pragma unroll
        for (int o = 16; o; o >>= 1) rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
      }
      const long long seg_start = it;
      for (; it < seg_end; ++it) {
        const int ct = ct_first + (int)(it - seg_start);  // a segment's column tiles are consecutive
        const int buf = BWD ? 0 : (tile_ctr & (kNB - 1));
        const int cb = ct * kColsPerTile + h * 128 + u * 64;  // global column of this thread's column 0
        const int igd = ig + p.row_off;  // the column holding this row's positive pair
        const bool diag_tile = (p.diag_on || p.self_mask) && igd >= cb && igd < cb + 64;
        const bool clean = row_ok && (cb + 64 <= p.ncols) && !diag_tile;
        // backward: G_ij = 2^{y-r2_i} + 2^{y-c2_j} = E (1 + p_i q_j) with E = 2^{y-r2_i}, p_i = 2^{r2_i-cmin},
        // q_j = 2^{cmin-c2_j} (cmin = the tile's smallest column LSE of this warp): one exponential per logit.
        // Valid while every r2_i - c2_j <= 60 (then a lost underflowed E carries a term < 2^-66); otherwise
        // (warp-uniform, rare) the tile takes both exponentials.  cval holds q (fast) or c2 (exact).
        float cmin = INFINITY;
        bool gfast = true;
        if (BWD) {  // publish this tile's column terms to the warp's slot, then prefetch the next tile's
          cmin = fminf(pc.x, pc.y);
#pragma unroll
          for (int o = 16; o; o >>= 1) cmin = fminf(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
          gfast = !(rmax - cmin > 60.f);
          const float2 cq = gfast ? make_float2(ex2(cmin - pc.x), ex2(cmin - pc.y)) : pc;
          *reinterpret_cast<float2*>(&cval[ep][2 * lane]) = cq;
          __syncwarp();
          if (it + 1 < seg_end) load_pc_ct(ct + 1);
          else if (it + 1 < nk) load_pc(it + 1);
        }
        // forward: the 2 warps of a group each merge 32 of its 64 columns into the slot (prefetched here)
        float2 pre = make_float2(-INFINITY, 0.f);
        const bool first_visit = !p.slots_merge && it < p.n_ct;
        float2* slot = p.col_slots + (long long)blockIdx.x * p.slot_ld;
        const int cm = cb + rh * 32 + lane;  // the column this lane merges
        if (!BWD && !first_visit && cm < p.ncols) pre = slot[cm];
        wc.wait(&sfull[buf], (sph >> buf) & 1u, 8);
        sph ^= 1u << buf;
        tc_fence_after();
        float v[64];
        if constexpr (BWD) {  // 32x32b: thread = one row, 64 consecutive columns
          tmem_ld32(laddr + buf * 128, v);
          tmem_ld32(laddr + buf * 128 + 32, v + 32);
        } else {  // 16x256b: thread = 4 rows x 16 columns (see forward statistics below)
          tmem_ld16x256x8(laddr + buf * 128, v);
          tmem_ld16x256x8(laddr + (16u << 16) + buf * 128, v + 32);
        }
        tmem_ld_wait();
        if constexpr (BWD) {  // single S buffer: each warp releases it as soon as its slice is in registers
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(&sfree[buf], 0);
        }

        if (DBG && p.noepi) {
          if (!BWD) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&sfree[buf], 0);
          } else {
            wc.wait(&gfree, gfph ^ 1, 9);
            gfph ^= 1;
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&gready, 0);
          }
        } else if constexpr (!BWD) {
          // ---------------------------------------------------------- forward statistics
          // 16x256b layout: t0 = lane & 3, t1 = lane >> 2; value v[eta*32 + rho*4 + kap*2 + c] is
          //   row  32*rh + 16*eta + 8*kap + t1 (of this CTA's 64),  column cb + 8*rho + 2*t0 + c.
          // Row references are thread-local maxima (any upper bound works for shared exponentials), so rows
          // need no shuffles; column sums reduce 4 rows in-thread, then 8 lanes (3 butterfly rounds).
          const int rowbase = rb * kRowsPerPair + (int)cta * 64 + rh * 32 + (lane >> 2);
          const float4 cs = fwd_chunk_stats<true>(v, laddr + buf * 128, rowbase, cb, p, lane, mrow, srow);
          const float m0 = cs.x, S0 = cs.y, m1 = cs.z, S1 = cs.w;
          // release this S buffer (per warp) only after the (rare) exact fallback has re-read it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(&sfree[buf], 0);
          // xch is double-buffered by tile parity: a warp can only rewrite buffer t&1 at tile t+2 after
          // passing tile t+1's barrier, i.e. after its partner finished reading tile t
          float2(*xb)[2][64] = xch[tile_ctr & 1];
          *reinterpret_cast<float4*>(&xb[grp][rh][2 * lane]) = make_float4(m0, S0, m1, S1);
          named_bar_sync(2 + grp, 64);
          {
            float2 a = merge2(xb[grp][0][rh * 32 + lane], xb[grp][1][rh * 32 + lane]);
            if (!first_visit) a = merge2(pre, a);
            if (cm < p.ncols) slot[cm] = a;
          }
        } else {
          // ---------------------------------------------------------- backward: G tile -> smem (bf16)
          const float* cv = cval[ep];
          uint32_t pk[32];
          if (gfast) {
            const float pr = ex2(r2 - cmin);
            const float2 kk = make_float2(k2, k2), nr = make_float2(-r2, -r2), pp = make_float2(pr, pr);
#pragma unroll
            for (int j = 0; j < 64; j += 4) {
              const float4 q4 = *reinterpret_cast<const float4*>(cv + j);
              const float2 t0 = __ffma2_rn(make_float2(v[j + 0], v[j + 1]), kk, nr);
              const float2 t1 = __ffma2_rn(make_float2(v[j + 2], v[j + 3]), kk, nr);
              const float2 e0 = make_float2(ex2(t0.x), ex2(t0.y)), e1 = make_float2(ex2(t1.x), ex2(t1.y));
              const float2 g0 = INFCL_MUTATION == 2 ? e0 : __ffma2_rn(e0, __fmul2_rn(pp, make_float2(q4.x, q4.y)), e0);
              const float2 g1 = __ffma2_rn(e1, __fmul2_rn(pp, make_float2(q4.z, q4.w)), e1);
              pk[j / 2] = pack_bf16(g0.x, g0.y);
              pk[j / 2 + 1] = pack_bf16(g1.x, g1.y);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 64; j += 4) {
              const float4 c4 = *reinterpret_cast<const float4*>(cv + j);
              const float g0 = ex2(fmaf(v[j + 0], k2, -r2)) + ex2(fmaf(v[j + 0], k2, -c4.x));
              const float g1 = ex2(fmaf(v[j + 1], k2, -r2)) + ex2(fmaf(v[j + 1], k2, -c4.y));
              const float g2 = ex2(fmaf(v[j + 2], k2, -r2)) + ex2(fmaf(v[j + 2], k2, -c4.z));
              const float g3 = ex2(fmaf(v[j + 3], k2, -r2)) + ex2(fmaf(v[j + 3], k2, -c4.w));
              pk[j / 2] = pack_bf16(g0, g1);
              pk[j / 2 + 1] = pack_bf16(g2, g3);
            }
          }
          if (!clean) {  // ragged columns, invalid row, or the diagonal (added exactly in fp32 later)
#pragma unroll
            for (int j = 0; j < 64; j += 2) {
              const int jg = cb + j;
              const bool dm = p.diag_on || p.self_mask;  // positive (added exactly later) or self (excluded)
              const bool ok0 = row_ok && jg < p.ncols && !(dm && jg == igd);
              const bool ok1 = row_ok && jg + 1 < p.ncols && !(dm && jg + 1 == igd);
              pk[j / 2] &= (ok0 ? 0x0000FFFFu : 0u) | (ok1 ? 0xFFFF0000u : 0u);
            }
          }
          if constexpr (GC) {
            // fused backward: before this warp rewrites its 32 rows x 64 columns of sG, its TMA store of the
            // previous tile must have read them
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
          }
          wc.wait(&gfree, gfph ^ 1, 9);
          gfph ^= 1;
          const uint32_t gb = smem_u32(sG) + (2 * h + u) * kBox + r * 128;
#pragma unroll
          for (int c16 = 0; c16 < 8; ++c16)
            st_shared_v4(gb + ((c16 ^ (r & 7)) << 4), pk[c16 * 4 + 0], pk[c16 * 4 + 1], pk[c16 * 4 + 2],
                         pk[c16 * 4 + 3]);
          fence_proxy_async_smem();
          __syncwarp();  // all G writes of this warp done (and cval reads before the next tile's rewrite)
          if (lane == 0) mbar_arrive_cluster(&gready, 0);
          if constexpr (GC) {
            // fused backward: lane 0 stores the warp's 32 x 64 G block to ring row ((g % ring) * gc_pp + t) * 128
            // + cta * 64 + 32 rh of step g = wave * n_ct + ct once the slot is free (gc_free_upto, kept by the
            // signal warp), and counts the previous tile's store in gc_written once it is complete; the signal warp
            // publishes ready[g].  The epilogue never waits on a gpu-scope release or acquire.
            if (lane == 0) {
              const int w = rb / p.gc_pp;
              const long long g = (long long)w * p.n_ct + ct;
              if (g > ld_volatile_shared(&gc_free_upto)) {
                const unsigned long long t0 = clock64();
                while (g > ld_volatile_shared(&gc_free_upto)) {
                  __nanosleep(64);
                  if (clock64() - t0 > INFCL_WATCHDOG_CYCLES) watchdog_fire(13, (uint32_t)g);
                }
              }
              const int grow = (int)((g % p.gc_ring) * p.gc_pp + (rb - w * p.gc_pp)) * kRowsPerPair + (int)cta * 64;
              if (p.gc_hint & 2)
                tma_store_2d_hint(&tmGs, sG + (2 * h + u) * kBox + rh * 4096, h * 128 + u * 64, grow + rh * 32,
                                  policy_evict_last());
              else
                tma_store_2d(&tmGs, sG + (2 * h + u) * kBox + rh * 4096, h * 128 + u * 64, grow + rh * 32);
              bulk_commit();
              if (tile_ctr > 0) {
                bulk_wait<1>();
                red_release_cta_shared_add(&gc_written, 1u);
              }
            }
          }
        }
        ++tile_ctr;
      }
      if constexpr (!BWD) {
        // merge each row's 4 lane slices (t0), then its 4 column slices (h, u); write the segment's row partial
        const int t0 = lane & 3, t1 = lane >> 2;
#pragma unroll
        for (int ri = 0; ri < 4; ++ri) {
          float2 a = make_float2(mrow[ri], srow[ri]);
#pragma unroll
          for (int o = 1; o <= 2; o <<= 1) {
            float2 bq;
            bq.x = __shfl_xor_sync(0xffffffffu, a.x, o);
            bq.y = __shfl_xor_sync(0xffffffffu, a.y, o);
            a = merge2(a, bq);
          }
          if (t0 == 0) rowx[grp][rh * 32 + 16 * (ri >> 1) + 8 * (ri & 1) + t1] = a;
        }
        named_bar_sync(1, 256);
        if (grp == 0 && row_ok) {
          float2 a = merge2(merge2(rowx[0][r], rowx[1][r]), merge2(rowx[2][r], rowx[3][r]));
          p.row_parts[S.seg_slot(rb) * kRowsPerPair + cta * 64 + r] = a;
        }
        named_bar_sync(1, 256);
      } else {
        // drain dA^T: lanes = 128 d-rows of each 256-chunk, columns u*64.. = pair rows -> red.add into dA
        wc.wait(&dafull, daph, 10);
        daph ^= 1;
        tc_fence_after();
        const int row0 = rb * kRowsPerPair + u * 64;
        // a tail row block split between pairs goes to this pair's scratch slot (plain stores) and is added to
        // dA in pair order by tail_combine_kernel: every element gets its partials in a fixed order
        const bool tail_rb = p.tail_scratch != nullptr && rb >= S.W * S.P;
        float* tdst = tail_rb ? p.tail_scratch + (long long)(S.pair + rb - S.W * S.P) * kRowsPerPair * p.d_out +
                                    (long long)(u * 64) * p.d_out
                              : nullptr;
        for (int tc = 0; tc < p.NDC; ++tc) {
          const int d = tc * 256 + (int)cta * 128 + q * 32 + lane;
          for (int c = 0; c < 2; ++c) {
            float y[32];
            tmem_ld32(laddr + 128 + tc * 128 + c * 32, y);
            tmem_ld_wait();
            if (d < p.d_out) {
              if (tail_rb) {
#pragma unroll
                for (int i = 0; i < 32; ++i) tdst[(long long)(c * 32 + i) * p.d_out + d] = coef * y[i];
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (row0 + c * 32 + i < p.nrows)
                    red_add_f32(p.dA + (long long)(row0 + c * 32 + i) * p.ld_dA + d, coef * y[i]);
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&dafree, 0);
      }
    }
    if constexpr (GC) {
      if (lane == 0 && tile_ctr > 0) {
        bulk_wait<0>();
        red_release_cta_shared_add(&gc_written, 1u);
      }
    }
    wc.flush(2 + (ep & 1));
  }
  __syncwarp();
  if (DBG && p.dbg && threadIdx.x == 0) atomicAdd(p.dbg + 4 * 16 + 15, (unsigned long long)(clock64() - t_start));
  tc_fence_before();
  cluster_sync();
  if (warp == kWarpMMA) tmem_dealloc<2>(tbase, kTmemCols);
}

// ------------------------------------------------------------------------------------------ host side
PassGeom pass_geom(int nrows, int ncols) {
  PassGeom g;
  g.rpp = kRowsPerPair;
  g.n_rb = (nrows + kRowsPerPair - 1) / kRowsPerPair;
  g.n_ct = (ncols + kColsPerTile - 1) / kColsPerTile;
  g.n_items = (long long)g.n_rb * g.n_ct;
  const int pairs = max_pairs();
  g.npairs = (int)std::min<long long>(pairs, g.n_items);
  return g;
}

// Fused backward plan (GC): the split of the npairs CTA pairs into gc_pp producers and npairs - gc_pp consumers
// balances ceil(n_rb / pp) waves x n_ct producer tiles (each S + G + dA, ~ratio x a consumer tile's time) against
// each consumer's ceil(n_ct / pc) column tiles x n_rb consumer tiles; ring = steps resident in the G ring (a
// consumer holds its step's slot while it streams the step's pp tiles, so ~pc steps are live at a time).
GcPlan gc_plan(int nrows, int ncols, int dk) {
  GcPlan q{};
  static const bool off = [] {
    const char* e = getenv("INFCL_FUSED_BWD");
    return e && atoi(e) == 0;
  }();
  const PassGeom g = pass_geom(nrows, ncols);
  // below ~16K rows per launch the producer / consumer pipeline's fill and drain cost more than the saved S
  // recompute (virtual ring at cfg2, final round-2 build with the consumer tie-break: n = 4 (b_s = 16384) 12.7 ms
  // fused vs 14.7 two-pass, n = 8 (b_s = 8192) 18.3 vs 18.1; earlier builds crossed over at 32K rows);
  // INFCL_GC_MIN_ROWS overrides (tests force the fused kernel at small shapes)
  long long min_rows = 16384;
  if (const char* e = getenv("INFCL_GC_MIN_ROWS")) min_rows = atoll(e);
  if (off || dk > kMaxD || g.npairs < 2 || nrows < min_rows) return q;
  const int nparts = dk > 512 ? 2 : 1;  // consumer units per column tile (weights 2 : 1 when split)
  // producer tile time in consumer-chunk units x NDC (2.2 at d = 512 and 768): consumer-count sweeps of the final
  // round-2 build (profiles/gc_split_r02.log) put the optimum at 22 (b = 65536) and 23 (b = 262144) consumers at
  // d = 512, 25-27 (b = 65536) and 23 (b = 262144) at d = 768
  double ratio = 2.2;
  if (const char* e = getenv("INFCL_GC_RATIO")) ratio = std::max(0.1, atof(e));
  int best_pc = 1;
  double best = 1e300;
  const int NDC = (dk + 255) / 256;
  for (int pc = 1; pc < g.npairs; ++pc) {
    // two parts per column tile: an odd consumer count gives every consumer the same mix of both parts
    if (nparts == 2 && pc % 2 == 0) continue;
    const int pp = g.npairs - pc;
    // producer tile ~ ratio consumer tiles of NDC d chunks; a consumer's units cover ~NDC / pc of every column tile
    const double prod = (double)((g.n_rb + pp - 1) / pp) * g.n_ct * ratio * NDC;
    // consumers take the items round-robin: ceil(items / pc) items of ~n_rb / waves tiles x NDC / nparts chunks
    const int waves = (g.n_rb + pp - 1) / pp;
    const long long items = (long long)waves * g.n_ct * nparts;
    const double cons = (double)((items + pc - 1) / pc) * ((double)g.n_rb / waves) * ((double)NDC / nparts);
    const double cost = std::max(prod, cons);
    // ties go to MORE consumers: a producer that does not remove a wave only shortens the last one, while each extra
    // consumer lightens every wave's dT work (cfg2: 22 consumers 10.67 ms vs 21 11.19 ms, medians of 4 x 7 steps,
    // scripts/experiments/gc_split_ab.sh)
    if (cost <= best + 1e-9) {
      best = cost;
      best_pc = pc;
    }
  }
  if (const char* e = getenv("INFCL_GC_CONSUMERS")) best_pc = std::max(1, std::min(g.npairs - 1, atoi(e)));
  if (best >= 1e300 && !getenv("INFCL_GC_CONSUMERS")) return q;  // no admissible split (2 pairs, 2 parts)
  q.npairs = g.npairs;
  q.pc = best_pc;
  q.pp = g.npairs - best_pc;
  q.n_steps = (long long)((g.n_rb + q.pp - 1) / q.pp) * g.n_ct;
  // P_c + 4 steps: a smaller ring stays in L2 longer (G ring depth sweeps, profiles/gc_split_r02.log: b = 262144
  // P_c + 1..4 178-179 ms vs P_c + 11 185 ms; cfg2 and d = 768 within the run-to-run spread or slightly better)
  long long ring = q.pc + 4;
  // >= 2: a store warp signals step g - 1 only after storing step g, which waits for step g - ring to be read
  if (const char* e = getenv("INFCL_GC_RING")) ring = std::max(2, atoi(e));
  q.ring = (int)std::min<long long>(ring, q.n_steps);
  q.n_ctr = (q.pp + 1) * q.n_steps + (long long)g.n_ct * nparts;  // ready, consumed, unit_done
  q.ctr_bytes = ((size_t)q.n_ctr * sizeof(uint32_t) + 1023) / 1024 * 1024;
  q.bytes = q.ctr_bytes + (size_t)q.ring * q.pp * kRowsPerPair * kColsPerTile * 2;
  q.ok = true;
  return q;
}

template <bool BWD, bool GC>
static infcl_status launch_pair(const PassArgs& a, cudaStream_t s) {
  if (a.dk > kMaxD) return fail(INFCL_ERR_SHAPE, "feature dim above kernel limit 768");
  const PassGeom g = pass_geom(a.nrows, a.ncols);
  KParams k{};
  k.nrows = a.nrows;
  k.ncols = a.ncols;
  k.dk = a.dk;
  k.KB = (a.dk + 63) / 64;
  // ring stages hold two 16-KB boxes (8 MMAs per barrier round trip). Measured (DESIGN.md perf log): 16-KB
  // stages keep more bytes in flight in the forward but are 30 % slower -- the per-stage round trip dominates
  k.sbox = 2;
  if (const char* e = getenv("INFCL_SBOX"); e && !BWD) k.sbox = atoi(e) == 1 ? 1 : 2;  // A/B diagnostic
  k.stage_bytes = k.sbox * kBoxB;
  k.KC = k.sbox == 2 ? (k.KB + 1) / 2 : k.KB;
  k.NDC = (a.dk + 255) / 256;
  k.n_rb = g.n_rb;
  k.n_ct = g.n_ct;
  k.npairs = g.npairs;
  k.n_items = g.n_items;
  // s log2 e; never 0: at s = 0 the epilogues' masked -inf logits would give -inf * 0 = NaN, while FLT_MIN maps every
  // finite logit to 0 (flushed) exactly as s = 0 does
  k.k2 = std::max(a.scale * 1.4426950408889634f, 1.17549435e-38f);
  k.scale = a.scale;
  k.diag_on = a.diag_on;
  k.self_mask = a.self_mask;
  k.row_off = a.row_off;
  k.slots_merge = a.slots_merge;
  k.col_slots = a.col_slots;
  k.slot_ld = a.slot_ld;
  k.row_parts = a.row_parts;
  k.diag_out = a.diag_out;
  k.lse_row2 = a.lse_row2;
  k.lse_col2 = a.lse_col2;
  k.dA = a.dA;
  k.ld_dA = a.ld_dA;
  k.d_out = a.d_out;
  k.grad = a.grad;
  k.coef_base = a.coef_base;
  // deterministic tail: only where the last wave splits row blocks between pairs (never in the fused kernel,
  // whose tail row blocks are whole)
  k.tail_scratch = (BWD && !GC && a.tail_scratch && g.n_rb % g.npairs != 0) ? a.tail_scratch : nullptr;
  GcPlan q{};
  if (GC) {
    q = gc_plan(a.nrows, a.ncols, a.dk);
    // a workspace sized for another launch shape (the host entry's row blocks) holds fewer ring steps: the ring
    // depth only has to stay >= 2
    if (q.ok && a.gc_ws && a.gc_ws_bytes < q.bytes && a.gc_ws_bytes > q.ctr_bytes) {
      const size_t step_bytes = (size_t)q.pp * kRowsPerPair * kColsPerTile * 2;
      q.ring = (int)std::min<long long>(q.ring, (long long)((a.gc_ws_bytes - q.ctr_bytes) / step_bytes));
      q.bytes = q.ctr_bytes + (size_t)q.ring * step_bytes;
    }
    if (!q.ok || q.npairs != g.npairs || !a.gc_ws || a.gc_ws_bytes < q.bytes || q.ring < 2 || !a.dB)
      return fail(INFCL_ERR_INVALID_ARG, "fused backward: no plan or workspace");
    k.gc_pp = q.pp;
    k.gc_hint = 5;  // consumer G loads evict_first, A loads evict_last: -16 % energy per backward (measured)
    if (const char* e = getenv("INFCL_GC_HINT")) k.gc_hint = atoi(e);
    k.gc_ring = q.ring;
    k.g_ready = reinterpret_cast<uint32_t*>(a.gc_ws);
    k.g_consumed = k.g_ready + q.n_steps * q.pp;
    k.g_unit_done = k.g_consumed + q.n_steps;
    k.g_ring = reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(a.gc_ws) + q.ctr_bytes);
    k.dB = a.dB;
    k.ld_dB = a.ld_dB;
  }
  unsigned long long* dbg_buf = debug_buffer(s);
  const bool dbg_on = dbg_buf != nullptr;
  k.dbg = dbg_buf;
  // dynamic smem starts after the static part rounded up to 1024 B (the extern array's alignment)
  static int static_smem = -1;
  if (static_smem < 0) {
    cudaFuncAttributes fa;
    INFCL_CUDA_TRY(cudaFuncGetAttributes(&fa, pair_kernel<BWD, false, GC>));
    static_smem = (int)fa.sharedSizeBytes;
  }
  const long long budget = 232448 - ((static_smem + 1023) / 1024) * 1024;
  const size_t fixed = (size_t)k.KB * kBox + (BWD ? 4 * kBox : 0);
  int ns = (int)((budget - (long long)fixed) / k.stage_bytes);
  ns = std::min(ns, kMaxStages);
  if (const char* e = getenv("INFCL_STAGES")) ns = std::max(2, std::min(ns, atoi(e)));
  if (ns < 2) return fail(INFCL_ERR_SHAPE, "feature dim too large for the smem budget");
  k.n_stages = ns;
  k.pair_commit = (ns % 2 == 0 && !getenv("INFCL_NO_PAIR_COMMIT")) ? 1 : 0;
  const size_t smem = fixed + (size_t)ns * k.stage_bytes;
  if (GC) {  // consumers: one ring of 32-KB stages in the same dynamic smem
    k.n_stages_c = std::min((int)(smem / 32768) - 1, kMaxStages);  // + 32 KB: the drain's staging boxes
    if (k.n_stages_c < 2) return fail(INFCL_ERR_SHAPE, "fused backward: smem too small for the consumer ring");
  }

  CUtensorMap tmA, tmB, tmG, tmI, tmGs, tmDT;
  infcl_status st = make_tmap_bf16(&tmA, a.A, a.nrows, a.dk, a.ld, 64, 64);
  if (st) return st;
  if ((st = make_tmap_bf16(&tmB, a.B, a.ncols, a.dk, a.ld, 64, 128))) return st;
  if (GC) {
    if ((st = make_tmap_bf16(&tmG, static_cast<uint8_t*>(a.gc_ws) + q.ctr_bytes,
                             (uint64_t)q.ring * q.pp * kRowsPerPair, kColsPerTile, kColsPerTile, 64, 64)))
      return st;
    if ((st = make_tmap_bf16(&tmI, a.A, a.nrows, a.dk, a.ld, 64, 128))) return st;
    if ((st = make_tmap_bf16(&tmGs, static_cast<uint8_t*>(a.gc_ws) + q.ctr_bytes,
                             (uint64_t)q.ring * q.pp * kRowsPerPair, kColsPerTile, kColsPerTile, 64, 32)))
      return st;
    if ((st = make_tmap_f32_sw128(&tmDT, a.dB, a.ncols, a.d_out, a.ld_dB, 32, 32))) return st;
  } else {
    tmG = tmA;
    tmI = tmA;
    tmGs = tmA;
    tmDT = tmA;
  }

  k.noepi = !GC && getenv("INFCL_DEBUG_NOEPI") != nullptr;
  k.notma = !GC && getenv("INFCL_DEBUG_NOTMA") != nullptr;
  auto kern = dbg_on ? pair_kernel<BWD, true, GC> : pair_kernel<BWD, false, GC>;
  INFCL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int nthreads = GC ? kThreadsGC : kThreads;
  if (GC) {
    // producers and consumers wait on each other: every CTA pair must be resident at once
    static int max_clusters = -1;
    if (max_clusters < 0) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(2 * g.npairs);
      cfg.blockDim = dim3(nthreads);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      INFCL_CUDA_TRY(cudaOccupancyMaxActiveClusters(&max_clusters, (void*)kern, &cfg));
    }
    if (max_clusters < g.npairs)
      return fail(INFCL_ERR_UNSUPPORTED, "fused backward: only " + std::to_string(max_clusters) +
                                             " CTA pairs co-resident, need " + std::to_string(g.npairs));
    INFCL_CUDA_TRY(cudaMemsetAsync(a.gc_ws, 0, (size_t)q.n_ctr * sizeof(uint32_t), s));
  }
  cudaEvent_t e0 = profile_begin(s);
  kern<<<dim3(2 * g.npairs), dim3(nthreads), smem, s>>>(tmA, tmB, tmG, tmI, tmGs, tmDT, k);
  INFCL_CUDA_TRY(cudaGetLastError());
  profile_end(BWD ? 1 : 0, e0, s);
  if (k.tail_scratch) launch_tail_combine(k.tail_scratch, a.dA, a.ld_dA, a.nrows, a.d_out, g, s);
  if (dbg_on) debug_report(GC ? "BWD(fused)" : BWD ? "BWD" : "FWD", g.npairs, s, GC ? q.pp : g.npairs);
  ++launch_counter();
  return INFCL_OK;
}

infcl_status launch_pair_forward(const PassArgs& a, cudaStream_t s) {
  if (wide_forward_enabled()) return launch_wide_forward(a, s);
  return launch_pair<false, false>(a, s);
}

PassGeom fwd_geom(int nrows, int ncols) { return wide_forward_enabled() ? wide_geom(nrows, ncols) : pass_geom(nrows, ncols); }

cudaEvent_t profile_begin(cudaStream_t s) {
  if (!prof().on) return nullptr;
  cudaEvent_t e0;
  cudaEventCreate(&e0);
  cudaEventRecord(e0, s);
  return e0;
}
void profile_end(int kind, cudaEvent_t e0, cudaStream_t s) {
  if (!e0) return;
  cudaEvent_t e1;
  cudaEventCreate(&e1);
  cudaEventRecord(e1, s);
  prof().ev[kind].push_back({e0, e1});
}

static unsigned long long*& dbg_ptr() {
  static unsigned long long* b = nullptr;
  return b;
}
unsigned long long* debug_buffer_ptr() { return dbg_ptr(); }
unsigned long long* debug_buffer(cudaStream_t s) {
  static const bool on = getenv("INFCL_DEBUG_WAITS") != nullptr;
  if (!on) return nullptr;
  if (!dbg_ptr()) cudaMalloc(&dbg_ptr(), 10 * 16 * sizeof(unsigned long long));
  cudaMemsetAsync(dbg_ptr(), 0, 10 * 16 * sizeof(unsigned long long), s);
  return dbg_ptr();
}
// debug only: per-role mean wait cycles per CTA (roles: 0 TMA, 1 MMA, 2/3 epilogue lanes)
void debug_report(const char* name, int npairs, cudaStream_t s, int prod_pairs) {
  unsigned long long* buf = dbg_ptr();
  unsigned long long h[160];
  cudaMemcpyAsync(h, buf, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (prod_pairs < 0) prod_pairs = npairs;
  const double nctas = 2.0 * prod_pairs, ncons = 2.0 * (npairs - prod_pairs);
  fprintf(stderr, "[infcl dbg] %s kernel: mean cycles/CTA total=%.0f\n", name, h[4 * 16 + 15] / (2.0 * npairs));
  const char* names[12] = {"LOOP", "empty", "afree", "dafree", "gready", "full", "afull", "sfree", "sfull", "gfree",
                           "dafull/sfull-commit", "S-issue"};
  for (int role = 0; role < 4; ++role)
    for (int t = 0; t < 12; ++t)
      if (h[role * 16 + t])
        fprintf(stderr, "[infcl dbg]   role %d wait %-7s %12.0f\n", role, names[t],
                h[role * 16 + t] / (role >= 2 ? nctas * 4 : (role == 1 ? nctas / 2 : nctas)));
  if (prod_pairs == npairs) return;
  // fused backward: consumer TMA (5), consumer MMA (6), consumer drain warps (7), producer G store warp (8)
  const char* cn[4][12] = {
      {"ready-spin", "empty", "", "", "", "", "", "", "", "", "", ""},
      {"LOOP", "", "", "dafree", "full(G)", "full(A)", "", "", "", "", "", ""},
      {"", "", "", "", "", "", "drain", "", "", "", "dafull", ""},
      {"", "gstore", "consumed-spin", "read-wait", "", "", "", "", "", "", "", ""}};
  const double norm[4] = {ncons, ncons / 2, ncons * 8, nctas};
  for (int role = 5; role < 9; ++role)
    for (int t = 0; t < 12; ++t)
      if (h[role * 16 + t])
        fprintf(stderr, "[infcl dbg]   %s %-13s %12.0f\n", role == 8 ? "store   " : role == 5 ? "c-TMA   " :
                role == 6 ? "c-MMA   " : "c-drain ", cn[role - 5][t], h[role * 16 + t] / norm[role - 5]);
}

void profile_enable(bool on) {
  prof_clear();
  prof().on = on;
}

infcl_status profile_read(int kind, int* launches, double* total_ms) {
  if (kind < 0 || kind > 2 || !launches || !total_ms) return fail(INFCL_ERR_INVALID_ARG, "bad profile query");
  double t = 0;
  for (auto& e : prof().ev[kind]) {
    INFCL_CUDA_TRY(cudaEventSynchronize(e.second));
    float ms = 0;
    INFCL_CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
    t += ms;
  }
  *launches = (int)prof().ev[kind].size();
  *total_ms = t;
  return INFCL_OK;
}
infcl_status launch_pair_backward(const PassArgs& a, cudaStream_t s) { return launch_pair<true, false>(a, s); }
infcl_status launch_pair_backward_fused(const PassArgs& a, cudaStream_t s) { return launch_pair<true, true>(a, s); }

}  // namespace infcl
