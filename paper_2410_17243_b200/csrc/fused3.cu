// Three-role fused backward (world 1, bf16, d <= 512; opt-in INFCL_BWD3=1, a measured negative result: see DESIGN.md
// section 5): Alg.4's single pass with every tensor-core instruction a 128-cycle M=256 N=256
// cta_group::2 MMA.  The CTA pairs split into
//   producers   [0, P)      S = s A_R B_C^T on 256-row x 256-column pair tiles (the wide forward's TMA/MMA loop),
//                           G_ij = 2^{y - r2_i} + 2^{y - c2_j} (Alg.4 l.10-11, Eq.7-8) -> bf16 -> G ring (TMA stores)
//   dI readers  [P, 2P)     reader p follows producer p: dI (256 rows x d) += G (256 x 256 j) B_C (256 j x d) over a
//                           row block's column tiles (Alg.4 l.12), accumulator in TMEM, drained once per row block
//   dT readers  [2P, n)     items (wave, column tile) round-robin: dT (256 j x d) += G^T A over the wave's tiles
//                           (Alg.4 l.13-15 without the per-tile read-modify-write of dT~)
// The G ring, its step counters and the drains are those of the two-role kernel (pair_kernel.cu, GC); here a ring
// tile is 256 rows x 256 columns (128 KB) and a step holds one tile per producer.  DESIGN.md section 5.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "host_utils.h"
#include "kernels.h"
#include "pair_common.cuh"
#include "ptx.cuh"

namespace infcl {

namespace {
constexpr int kR3 = 256;        // rows per producer tile (128 per SM)
constexpr int kStg3 = 32768;    // reader ring stage
constexpr int kWStage3 = 32768; // producer ring stage with streamed A: A block 16 KB + B block 16 KB
constexpr int kWarpSig3 = 10;   // producer signal warp
constexpr int kThreads3 = 352;

// tile t of step g = wave * n_ct + ct lives at ring rows ((g % ring) * P + t) * 256
__device__ __forceinline__ int ring_row3(long long g, int t, const KParams& p) {
  return (int)(((g % p.gc_ring) * p.gc_pp + t) * kR3);
}

// drain one 32 (TMEM lanes) x 32 (columns) fp32 block through this warp's 4-KB staging box (128-B swizzle) and a
// TMA reduce-add at tensor coordinates (c0 = feature, c1 = row of dst)
__device__ __forceinline__ void drain_block(const CUtensorMap* tm, uint8_t* stg_ptr, uint32_t stg, int lane,
                                            const float (&y)[32], float coef, int c0, int c1) {
  if (lane == 0) bulk_wait_read<0>();
  __syncwarp();
#pragma unroll
  for (int c4 = 0; c4 < 8; ++c4)
    st_shared_v4f(stg + lane * 128 + ((c4 ^ (lane & 7)) << 4), coef * y[4 * c4], coef * y[4 * c4 + 1],
                  coef * y[4 * c4 + 2], coef * y[4 * c4 + 3]);
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_reduce_add_2d(tm, stg_ptr, c0, c1);
    bulk_commit();
  }
}
}  // namespace

// DBG (INFCL_DEBUG_WAITS): per-role wait cycles into p.dbg[role * 16 + slot] (roles: producer TMA 0, MMA 1,
// epilogue 2; dI reader TMA 4, MMA 5, drain 6; dT reader TMA 7, MMA 8, drain 9)
#define W3(SLOT, ...)                                            \
  do {                                                           \
    const unsigned long long _t0 = DBG ? clock64() : 0ull;       \
    __VA_ARGS__;                                                 \
    if (DBG) dacc[SLOT] += clock64() - _t0;                      \
  } while (0)

template <bool RESA, bool DBG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads3, 1)
    bwd3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmG2,
                const __grid_constant__ CUtensorMap tmGs, const __grid_constant__ CUtensorMap tmDT,
                const __grid_constant__ CUtensorMap tmDI, const __grid_constant__ KParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u)) __trap();
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], sfull[2], sfree[2], dafull, dafree;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float cval[8][64];  // producer: each warp's 64 column terms (q_j or c2_j) of a chunk
  __shared__ long long gc_free_upto;
  __shared__ uint32_t gc_written;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int P = p.gc_pp;
  const int role = pair < P ? 0 : pair < 2 * P ? 1 : 2;  // producer, dI reader, dT reader
  const int NS = role == 0 ? p.n_stages : p.n_stages_c;
  // producers and dI readers walk the same schedule: producer p's row blocks, all column tiles each
  const Sched S(p.n_rb, p.n_ct, P, role == 1 ? pair - P : pair, true);
  const long long nk = role <= 1 ? S.n_local() : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], 1);
      mbar_init(&sfree[b], 16);
    }
    mbar_init(&dafull, 1);
    mbar_init(&dafree, 16);
    gc_free_upto = (long long)p.gc_ring - 1;
    gc_written = 0;
    fence_mbar_init();
  }
  if (warp == kWarpTMA && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (role == 0) tma_prefetch_desc(&tmGs);
    if (role == 1) {
      tma_prefetch_desc(&tmG2);
      tma_prefetch_desc(&tmDI);
    }
    if (role == 2) {
      tma_prefetch_desc(&tmG);
      tma_prefetch_desc(&tmDT);
    }
  }
  if (warp == kWarpMMA) tmem_alloc<2>(&tmem_base, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t nparts_u = 1;
  const float coef = p.coef_base * __ldg(p.grad);
  unsigned long long dacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const unsigned long long t_begin = DBG ? clock64() : 0ull;
  int drole = -1;  // this thread's role slot for the debug flush (lane 0 of a timed warp)

  if (role == 0) {
    // ======================================================================================== producers
    uint8_t* sA = smem_raw;
    uint8_t* sStg = smem_raw + (RESA ? p.KB * kBoxB : 0);                    // epilogue staging, 8 x 4 KB
    uint8_t* sStage = sStg + 8 * 4096;
    constexpr int kStg = RESA ? kBoxB : kWStage3;
    if (warp == kWarpTMA) {
      drole = 0;
      if (lane == 0) {
        int stage = 0;
        uint32_t ph = 0;
        long long it = 0;
        while (it < nk) {
          int rb, ct0;
          S.decode(it, rb, ct0);
          const long long seg_end = S.seg_end(it), seg_start = it;
          const int a_row = rb * kR3 + (int)cta * 128;
          for (int ct = ct0; it < seg_end; ++it, ++ct) {
            const int b_row = ct * kColsPerTile + (int)cta * 128;
            const bool lda = !RESA || it == seg_start;
            for (int kb = 0; kb < p.KB; ++kb) {
              if (!p.pair_commit || !(stage & 1)) W3(1, mbar_wait(&empty[stage], ph ^ 1, 1));
              if (cta == 0) mbar_arrive_expect_tx(&full[stage], (lda ? 4 : 2) * kBoxB);
              uint8_t* dst = sStage + stage * kStg;
              if (lda) tma_load_2d_pair(RESA ? sA + kb * kBoxB : dst, &tmA, &full[stage], kb * 64, a_row);
              tma_load_2d_pair(RESA ? dst : dst + kBoxB, &tmB, &full[stage], kb * 64, b_row);
              if (++stage == NS) {
                stage = 0;
                ph ^= 1;
              }
            }
          }
        }
      }
    } else if (warp == kWarpMMA) {
      drole = cta == 0 ? 1 : -1;
      if (cta == 0) {
        int stage = 0;
        uint32_t ph = 0, sfph = 0;
        const uint32_t idS = idesc_bf16(256, 256, 0, 0);
        for (long long it = 0; it < nk; ++it) {
          const int buf = (int)(it & 1);
          W3(3, mbar_wait_cluster(&sfree[buf], ((sfph >> buf) & 1u) ^ 1u, 7));
          sfph ^= 1u << buf;
          tc_fence_after();
          const uint32_t dS = tbase + buf * 256;
          for (int kb = 0; kb < p.KB; ++kb) {
            W3(5, mbar_wait(&full[stage], ph, 5));
            tc_fence_after();
            const uint32_t st = smem_u32(sStage + stage * kStg);
            const uint32_t sa = RESA ? smem_u32(sA + kb * kBoxB) : st;
            umma_stage_pair<false, 0, 0>(dS, (uint32_t)smem_desc_sw128(sa, 16, 1024),
                                         (uint32_t)smem_desc_sw128(RESA ? st : st + kBoxB, 16, 1024), idS, kb != 0);
            ring_release(empty, stage, p.pair_commit);
            if (++stage == NS) {
              stage = 0;
              ph ^= 1;
            }
          }
          umma_commit_pair_mc_warp(&sfull[buf], 0x3);
        }
      }
    } else if (warp == kWarpSig3) {
      // publishes each tile once its 16 chunk stores (8 warps x 2) completed; keeps the ring-slot horizon
      if (lane == 0) {
        const long long n_steps = (long long)((p.n_rb + P - 1) / P) * p.n_ct;
        // a step is read by its wave's dI readers (one per tile) and one dT reader
        auto readers = [&](long long g) { return (uint32_t)min(P, p.n_rb - (int)(g / p.n_ct) * P) + nparts_u; };
        long long fu = (long long)p.gc_ring - 1, k = 0;
        unsigned long long t_last = clock64();
        while (k < nk) {
          bool moved = false;
          while (fu + 1 < n_steps &&
                 ld_acquire_gpu(p.g_consumed + (fu + 1 - p.gc_ring)) >= readers(fu + 1 - p.gc_ring)) {
            ++fu;
            moved = true;
          }
          if (moved) st_volatile_shared(&gc_free_upto, fu);
          const uint32_t wr = ld_acquire_cta_shared(&gc_written);
          while (k < nk && wr >= 16u * (uint32_t)(k + 1)) {
            int rb, ct;
            S.decode(k, rb, ct);
            const int w = rb / P;
            fence_acq_rel_gpu();
            red_release_gpu_add(p.g_ready + ((long long)w * p.n_ct + ct) * P + (rb - w * P), 1u);
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
    } else if (warp < 8) {
      // epilogue: warp (q, u) = rows 32q + lane of this CTA's 128, columns 128u .. 128u + 127 in two 64-column chunks
      drole = 2;
      const int q = warp & 3, u = warp >> 2;
      const uint32_t laddr = tbase + ((uint32_t)(q * 32) << 16) + u * 128;
      uint8_t* stg_ptr = sStg + warp * 4096;
      const uint32_t stg = smem_u32(stg_ptr);
      const float k2 = p.k2;
      uint32_t sph = 0;
      int chunks = 0;
      // column LSEs (log2) of the next chunk, lane l: columns 2l, 2l + 1 of the chunk (+inf: no column)
      float2 pc;
      auto load_pc = [&](int col0) {
        const int j = col0 + 2 * lane;
        pc.x = j < p.ncols ? __ldg(p.lse_col2 + j) : INFINITY;
        pc.y = j + 1 < p.ncols ? __ldg(p.lse_col2 + j + 1) : INFINITY;
      };
      long long it = 0;
      if (nk > 0) {
        int rb0, ct0;
        S.decode(0, rb0, ct0);
        load_pc(ct0 * kColsPerTile + u * 128);
      }
      while (it < nk) {
        int rb, ct_first;
        S.decode(it, rb, ct_first);
        const long long seg_end = S.seg_end(it), seg_start = it;
        const int ig = rb * kR3 + (int)cta * 128 + q * 32 + lane;  // this thread's row
        const bool row_ok = ig < p.nrows;
        const float r2 = row_ok ? __ldg(p.lse_row2 + ig) : 0.f;
        float rmax = row_ok ? r2 : -INFINITY;
#pragma unroll
        for (int o = 16; o; o >>= 1) rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        const int w = rb / P, t = rb - w * P;
        for (; it < seg_end; ++it) {
          const int ct = ct_first + (int)(it - seg_start);
          const int buf = (int)(it & 1);
          const long long g = (long long)w * p.n_ct + ct;
          W3(6, mbar_wait(&sfull[buf], (sph >> buf) & 1u, 8));
          sph ^= 1u << buf;
          tc_fence_after();
#pragma unroll 1
          for (int ch = 0; ch < 2; ++ch) {
            const int cb = ct * kColsPerTile + u * 128 + ch * 64;
            // this chunk's column terms -> cval (shared by the warp's rows); then prefetch the next chunk's
            float cmin = fminf(pc.x, pc.y);
#pragma unroll
            for (int o = 16; o; o >>= 1) cmin = fminf(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
            const bool gfast = !(rmax - cmin > 60.f);
            const float2 cq = gfast ? make_float2(ex2(cmin - pc.x), ex2(cmin - pc.y)) : pc;
            *reinterpret_cast<float2*>(&cval[warp][2 * lane]) = cq;
            __syncwarp();
            if (ch == 0) {
              load_pc(cb + 64);
            } else if (it + 1 < nk) {
              int rbn, ctn;
              S.decode(it + 1, rbn, ctn);
              load_pc(ctn * kColsPerTile + u * 128);
            }
            float v[64];
            tmem_ld32(laddr + buf * 256 + ch * 64, v);
            tmem_ld32(laddr + buf * 256 + ch * 64 + 32, v + 32);
            tmem_ld_wait();
            if (ch == 1) {  // both chunks are in registers: the S buffer may be refilled
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(&sfree[buf], 0);
            }
            const float* cv = cval[warp];
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
                const float2 g0 = __ffma2_rn(e0, __fmul2_rn(pp, make_float2(q4.x, q4.y)), e0);
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
            const int igd = ig + p.row_off;  // the column of this row's positive pair
            const bool diag = p.diag_on && igd >= cb && igd < cb + 64;
            if (!row_ok || diag || cb + 64 > p.ncols) {  // ragged, invalid row, diagonal (added exactly in fp32)
#pragma unroll
              for (int j = 0; j < 64; j += 2) {
                const int jg = cb + j;
                const bool ok0 = row_ok && jg < p.ncols && !(p.diag_on && jg == igd);
                const bool ok1 = row_ok && jg + 1 < p.ncols && !(p.diag_on && jg + 1 == igd);
                pk[j / 2] &= (ok0 ? 0x0000FFFFu : 0u) | (ok1 ? 0xFFFF0000u : 0u);
              }
            }
            __syncwarp();  // every lane read cval before the next chunk rewrites it
            // stage the 32 x 64 block (SW128) and TMA-store it to the ring once the slot is free; count the
            // previous chunk's store once complete
            W3(7, if (lane == 0) bulk_wait_read<0>(); __syncwarp());
#pragma unroll
            for (int c16 = 0; c16 < 8; ++c16)
              st_shared_v4(stg + lane * 128 + ((c16 ^ (lane & 7)) << 4), pk[c16 * 4 + 0], pk[c16 * 4 + 1],
                           pk[c16 * 4 + 2], pk[c16 * 4 + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (g > ld_volatile_shared(&gc_free_upto)) {
                const unsigned long long t0 = clock64();
                if (DBG) dacc[9] += 1;
                while (g > ld_volatile_shared(&gc_free_upto)) {
                  __nanosleep(64);
                  if (clock64() - t0 > INFCL_WATCHDOG_CYCLES) watchdog_fire(13, (uint32_t)g);
                }
              }
              tma_store_2d(&tmGs, stg_ptr, u * 128 + ch * 64, ring_row3(g, t, p) + (int)cta * 128 + q * 32);
              bulk_commit();
              if (chunks > 0) {
                bulk_wait<1>();
                red_release_cta_shared_add(&gc_written, 1u);
              }
            }
            ++chunks;
          }
        }
      }
      if (lane == 0 && chunks > 0) {
        bulk_wait<0>();
        red_release_cta_shared_add(&gc_written, 1u);
      }
    }
  } else if (role == 1) {
    // ======================================================================================== dI readers
    // per tile: two G stages (this CTA's 128 rows x 128 columns j each: boxes [128 rows][64 j]) and, per G stage,
    // one B_C stage per 256-feature chunk (128 j x this CTA's 128 features); dI (rows x features) in TMEM
    // (lane = row, NDC x 256 columns), drained once per row block
    uint8_t* sStage = smem_raw;
    uint8_t* sStg = smem_raw + NS * kStg3;
    if (warp == kWarpTMA) {
      drole = 4;
      if (lane == 0) {
        int stage = 0;
        uint32_t ph = 0;
        auto acquire = [&]() -> uint8_t* {
          W3(1, mbar_wait(&empty[stage], ph ^ 1u, 1));
          if (cta == 0) mbar_arrive_expect_tx(&full[stage], 2 * kStg3);
          return sStage + stage * kStg3;
        };
        auto advance = [&]() {
          if (++stage == NS) {
            stage = 0;
            ph ^= 1;
          }
        };
        for (long long it = 0; it < nk; ++it) {
          int rb, ct;
          S.decode(it, rb, ct);
          const int w = rb / P, t = rb - w * P;
          const long long g = (long long)w * p.n_ct + ct;
          W3(2, spin_geq(p.g_ready + g * P + t, 2u, 14));
          fence_proxy_async_global();
          const int grow = ring_row3(g, t, p) + (int)cta * 128;
          for (int jh = 0; jh < 2; ++jh) {
            uint8_t* gd = acquire();
            tma_load_2d_pair(gd, &tmG2, &full[stage], jh * 128, grow);
            tma_load_2d_pair(gd + kBoxB, &tmG2, &full[stage], jh * 128 + 64, grow);
            advance();
            for (int tc = 0; tc < p.NDC; ++tc) {
              uint8_t* dst = acquire();
              const int d0 = tc * 256 + (int)cta * 128, j0 = ct * kColsPerTile + jh * 128;
              tma_load_2d_pair(dst, &tmB, &full[stage], d0, j0);
              tma_load_2d_pair(dst + kBoxB, &tmB, &full[stage], d0 + 64, j0);
              advance();
            }
          }
        }
      }
    } else if (warp == kWarpMMA) {
      drole = cta == 0 ? 5 : -1;
      if (cta == 0) {
        const uint32_t idI = idesc_bf16(256, 256, 0, 1);
        int stage = 0;
        uint32_t ph = 0, dph = 0;
        auto advance = [&]() {
          if (++stage == NS) {
            stage = 0;
            ph ^= 1;
          }
        };
        long long it = 0;
        while (it < nk) {
          int rb, ct0;
          S.decode(it, rb, ct0);
          const long long seg_end = S.seg_end(it), seg_start = it;
          W3(3, mbar_wait_cluster(&dafree, dph ^ 1u, 3));
          dph ^= 1;
          tc_fence_after();
          const int w = rb / P;
          for (int ct = ct0; it < seg_end; ++it, ++ct) {
            const long long g = (long long)w * p.n_ct + ct;
            for (int jh = 0; jh < 2; ++jh) {
              const int gs = stage;
              W3(4, mbar_wait(&full[gs], ph, 4));
              tc_fence_after();
              if (jh == 1 && lane == 0) red_release_gpu_add(p.g_consumed + g, 1u);  // this tile has been read
              __syncwarp();
              const uint32_t a_lo = (uint32_t)smem_desc_sw128(smem_u32(sStage + gs * kStg3), 16, 1024);
              advance();
              for (int tc = 0; tc < p.NDC; ++tc) {
                W3(5, mbar_wait(&full[stage], ph, 5));
                tc_fence_after();
                const uint32_t b_lo = (uint32_t)smem_desc_sw128(smem_u32(sStage + stage * kStg3), kBoxB, 1024);
                umma_stage_kmn_pair<(kBoxB >> 4)>(tbase + tc * 256, a_lo, b_lo, idI,
                                                  (it != seg_start || jh != 0) ? 1u : 0u);
                umma_commit_pair_mc_warp(&empty[stage], 0x3);
                advance();
              }
              umma_commit_pair_mc_warp(&empty[gs], 0x3);
            }
          }
          umma_commit_pair_mc_warp(&dafull, 0x3);
        }
      }
    } else if (warp < 8) {
      drole = 6;
      const int q = warp & 3, u = warp >> 2;
      uint8_t* stg_ptr = sStg + warp * 4096;
      const uint32_t stg = smem_u32(stg_ptr);
      uint32_t daph = 0;
      long long it = 0;
      while (it < nk) {
        int rb, ct0;
        S.decode(it, rb, ct0);
        it = S.seg_end(it);
        W3(6, mbar_wait_cluster(&dafull, daph, 10));
        daph ^= 1;
        tc_fence_after();
        const int row0 = rb * kR3 + (int)cta * 128 + q * 32;
        for (int tc = 0; tc < p.NDC; ++tc)
          for (int cc = 0; cc < 4; ++cc) {
            const int col0 = u * 128 + cc * 32;
            float y[32];
            tmem_ld32(tbase + ((uint32_t)(q * 32) << 16) + tc * 256 + col0, y);
            tmem_ld_wait();
            drain_block(&tmDI, stg_ptr, stg, lane, y, coef, tc * 256 + col0, row0);
          }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&dafree, 0);
      }
      if (lane == 0) bulk_wait<0>();
    }
  } else {
    // ======================================================================================== dT readers
    // items k = wave * n_ct + ct round-robin (reader c: k = c, c + C, ...); per tile two 128-row halves, each a G
    // stage (this CTA's 128 columns j x 128 rows: boxes (ib, jb) of 64 x 64) and one stage of A per chunk
    const int C = p.npairs - 2 * P, c = pair - 2 * P;
    const int nW = (p.n_rb + P - 1) / P;
    const long long nitems = (long long)nW * p.n_ct;
    uint8_t* sStage = smem_raw;
    uint8_t* sStg = smem_raw + NS * kStg3;
    if (warp == kWarpTMA) {
      drole = 7;
      if (lane == 0) {
        const uint64_t polG = policy_evict_first(), polA = policy_evict_last();
        int stage = 0;
        uint32_t ph = 0;
        auto acquire = [&]() -> uint8_t* {
          W3(1, mbar_wait(&empty[stage], ph ^ 1u, 1));
          if (cta == 0) mbar_arrive_expect_tx(&full[stage], 2 * kStg3);
          return sStage + stage * kStg3;
        };
        auto advance = [&]() {
          if (++stage == NS) {
            stage = 0;
            ph ^= 1;
          }
        };
        for (long long kk = c; kk < nitems; kk += C) {
          const int w = (int)(kk / p.n_ct), ct = (int)(kk % p.n_ct);
          const int nt = min(P, p.n_rb - w * P);
          const long long g = (long long)w * p.n_ct + ct;
          for (int t = 0; t < nt; ++t) {
            W3(2, spin_geq(p.g_ready + g * P + t, 2u, 14));
            fence_proxy_async_global();
            for (int h = 0; h < 2; ++h) {
              uint8_t* gd = acquire();
              const int grow = ring_row3(g, t, p) + h * 128;
#pragma unroll
              for (int ib = 0; ib < 2; ++ib)
#pragma unroll
                for (int jb = 0; jb < 2; ++jb)
                  tma_load_2d_pair_hint(gd + (2 * ib + jb) * kBox, &tmG, &full[stage], ((int)cta * 2 + jb) * 64,
                                        grow + ib * 64, polG);
              advance();
              const int r0 = (w * P + t) * kR3 + h * 128;
              for (int tc = 0; tc < p.NDC; ++tc) {
                uint8_t* dst = acquire();
                const int d0 = tc * 256 + (int)cta * 128;
                tma_load_2d_pair_hint(dst, &tmA, &full[stage], d0, r0, polA);
                tma_load_2d_pair_hint(dst + kBoxB, &tmA, &full[stage], d0 + 64, r0, polA);
                advance();
              }
            }
          }
        }
      }
    } else if (warp == kWarpMMA) {
      drole = cta == 0 ? 8 : -1;
      if (cta == 0) {
        const uint32_t idT = idesc_bf16(256, 256, 1, 1);
        int stage = 0;
        uint32_t ph = 0, dph = 0;
        auto advance = [&]() {
          if (++stage == NS) {
            stage = 0;
            ph ^= 1;
          }
        };
        for (long long kk = c; kk < nitems; kk += C) {
          const int w = (int)(kk / p.n_ct), ct = (int)(kk % p.n_ct);
          const int nt = min(P, p.n_rb - w * P);
          const long long g = (long long)w * p.n_ct + ct;
          W3(3, mbar_wait_cluster(&dafree, dph ^ 1u, 3));
          dph ^= 1;
          tc_fence_after();
          for (int t = 0; t < nt; ++t) {
            for (int h = 0; h < 2; ++h) {
              const int gs = stage;
              W3(4, mbar_wait(&full[gs], ph, 4));
              tc_fence_after();
              const uint32_t a_lo = (uint32_t)smem_desc_sw128(smem_u32(sStage + gs * kStg3), kBox, 1024);
              advance();
              for (int tc = 0; tc < p.NDC; ++tc) {
                W3(5, mbar_wait(&full[stage], ph, 5));
                tc_fence_after();
                const uint32_t b_lo = (uint32_t)smem_desc_sw128(smem_u32(sStage + stage * kStg3), kBoxB, 1024);
                umma_stage_dT_pair(tbase + tc * 256, a_lo, b_lo, idT, (t != 0 || h != 0) ? 1u : 0u);
                umma_commit_pair_mc_warp(&empty[stage], 0x3);
                advance();
              }
              umma_commit_pair_mc_warp(&empty[gs], 0x3);
            }
          }
          // every tile of step g is in smem: when the step's dI readers have read it too (as a rule, long before),
          // its ring lines are dead -- drop them without a write-back; then the slot may be refilled
          if (ld_acquire_gpu(p.g_consumed + g) >= (uint32_t)nt) {
            for (int t = 0; t < nt; ++t) {
              const uint16_t* tl = p.g_ring + (long long)ring_row3(g, t, p) * kColsPerTile;
#pragma unroll 4
              for (int i = 0; i < 32; ++i) discard_l2_line(tl + (i * 32 + lane) * 64);
            }
          }
          __syncwarp();
          if (lane == 0) red_release_gpu_add(p.g_consumed + g, 1u);
          umma_commit_pair_mc_warp(&dafull, 0x3);
        }
      }
    } else if (warp < 8) {
      drole = 9;
      const int q = warp & 3, u = warp >> 2;
      uint8_t* stg_ptr = sStg + warp * 4096;
      const uint32_t stg = smem_u32(stg_ptr);
      uint32_t daph = 0;
      for (long long kk = c; kk < nitems; kk += C) {
        const int w = (int)(kk / p.n_ct), ct = (int)(kk % p.n_ct);
        W3(6, mbar_wait_cluster(&dafull, daph, 10));
        daph ^= 1;
        tc_fence_after();
        // waves reach each dT element in wave order (bitwise reproducible): the column tile's previous wave has
        // completed all 16 drain warps' reductions
        if (w > 0) {
          if (lane == 0) {
            W3(8, spin_geq(p.g_unit_done + ct, 16u * (uint32_t)w, 17));
            fence_proxy_async_global();
          }
          __syncwarp();
        }
        const int j0 = ct * kColsPerTile + (int)cta * 128 + q * 32;
        for (int tc = 0; tc < p.NDC; ++tc)
          for (int cc = 0; cc < 4; ++cc) {
            const int col0 = u * 128 + cc * 32;
            float y[32];
            tmem_ld32(tbase + ((uint32_t)(q * 32) << 16) + tc * 256 + col0, y);
            tmem_ld_wait();
            drain_block(&tmDT, stg_ptr, stg, lane, y, coef, tc * 256 + col0, j0);
          }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cluster(&dafree, 0);
          bulk_wait<0>();
          red_release_gpu_add(p.g_unit_done + ct, 1u);
        }
      }
    }
  }
  if (DBG && p.dbg && lane == 0 && drole >= 0) {
    dacc[0] = clock64() - t_begin;
    for (int i = 0; i < 12; ++i)
      if (dacc[i]) atomicAdd(p.dbg + drole * 16 + i, dacc[i]);
    atomicAdd(p.dbg + drole * 16 + 15, 1ull);  // contributing threads
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == kWarpMMA) tmem_dealloc<2>(tbase, 512);
}

// ------------------------------------------------------------------------------------------ host side
// INFCL_DEBUG_WAITS: mean cycles per timed thread of each role's waits
static void debug_report3(int P, int C, cudaStream_t s) {
  unsigned long long h[160];
  cudaMemcpyAsync(h, debug_buffer_ptr(), sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  const char* rn[10] = {"prod-TMA", "prod-MMA", "prod-epi", "", "dI-TMA", "dI-MMA", "dI-drain", "dT-TMA", "dT-MMA",
                        "dT-drain"};
  const char* sn[12] = {"TOTAL", "empty", "ready-spin", "sfree/dafree", "full(G)", "full", "sfull/dafull",
                        "stage-read", "unit-spin", "slot-waits(n)", "", ""};
  fprintf(stderr, "[infcl dbg] bwd3: P=%d producers, %d dI readers, %d dT readers\n", P, P, C);
  for (int r = 0; r < 10; ++r) {
    const double n = (double)h[r * 16 + 15];
    if (n == 0) continue;
    for (int t = 0; t < 12; ++t)
      if (h[r * 16 + t]) fprintf(stderr, "[infcl dbg]   %-9s %-14s %12.0f\n", rn[r], sn[t], h[r * 16 + t] / n);
  }
}

Gc3Plan gc3_plan(int nrows, int ncols, int dk) {
  Gc3Plan q{};
  // opt-in (INFCL_BWD3=1): measured 5-8 % slower than the two-role kernel at cfg2;
  // INFCL_FUSED_BWD=0 (the two passes) wins over both
  static const bool on = [] {
    const char* e = getenv("INFCL_BWD3");
    const char* f = getenv("INFCL_FUSED_BWD");
    return (e && atoi(e) != 0) && !(f && atoi(f) == 0);
  }();
  if (!on || dk > 512) return q;
  const int n_rb = (nrows + kR3 - 1) / kR3, n_ct = (ncols + kColsPerTile - 1) / kColsPerTile;
  const int npairs = max_pairs();
  if (npairs < 3 || n_rb < 1) return q;
  // time per producer tile : dI tile : dT tile (256 rows) -- equal FLOPs; tunable (INFCL_BWD3_RATIO = p,i,t)
  double rp = 1.0, ri = 1.0, rt = 1.0;
  if (const char* e = getenv("INFCL_BWD3_RATIO")) sscanf(e, "%lf,%lf,%lf", &rp, &ri, &rt);
  double best = 1e300;
  int bestP = 0;
  for (int P = 1; 2 * P < npairs; ++P) {
    const int C = npairs - 2 * P;
    const int waves = (n_rb + P - 1) / P;
    const double prod = (double)waves * n_ct * std::max(rp, ri);
    const long long items = (long long)waves * n_ct;
    const double cons = (double)((items + C - 1) / C) * ((double)n_rb / waves) * rt;
    const double cost = std::max(prod, cons);
    if (cost < best - 1e-9) {
      best = cost;
      bestP = P;
    }
  }
  if (const char* e = getenv("INFCL_BWD3_P")) bestP = std::max(1, std::min((npairs - 1) / 2, atoi(e)));
  if (bestP < 1) return q;
  q.npairs = npairs;
  q.pp = bestP;
  q.pc = npairs - 2 * bestP;
  q.n_rb = n_rb;
  q.n_ct = n_ct;
  q.n_steps = (long long)((n_rb + bestP - 1) / bestP) * n_ct;
  long long ring = q.pc + 12;
  if (const char* e = getenv("INFCL_GC_RING")) ring = std::max(2, atoi(e));
  q.ring = (int)std::min<long long>(ring, q.n_steps);
  q.n_ctr = (q.pp + 1) * q.n_steps + n_ct;  // ready, consumed, unit_done
  q.ctr_bytes = ((size_t)q.n_ctr * sizeof(uint32_t) + 1023) / 1024 * 1024;
  q.bytes = q.ctr_bytes + (size_t)q.ring * q.pp * kR3 * kColsPerTile * 2;
  q.ok = true;
  return q;
}

infcl_status launch_bwd3(const PassArgs& a, cudaStream_t s) {
  const Gc3Plan q = gc3_plan(a.nrows, a.ncols, a.dk);
  if (!q.ok || !a.gc_ws || a.gc_ws_bytes < q.bytes || !a.dB)
    return fail(INFCL_ERR_INVALID_ARG, "3-role backward: no plan or workspace");
  KParams k{};
  k.nrows = a.nrows;
  k.ncols = a.ncols;
  k.dk = a.dk;
  k.KB = (a.dk + 63) / 64;
  k.NDC = (a.dk + 255) / 256;
  k.n_rb = q.n_rb;
  k.n_ct = q.n_ct;
  k.npairs = q.npairs;
  k.k2 = std::max(a.scale * 1.4426950408889634f, 1.17549435e-38f);
  k.scale = a.scale;
  k.diag_on = a.diag_on;
  k.row_off = a.row_off;
  k.lse_row2 = a.lse_row2;
  k.lse_col2 = a.lse_col2;
  k.dA = a.dA;
  k.ld_dA = a.ld_dA;
  k.d_out = a.d_out;
  k.grad = a.grad;
  k.coef_base = a.coef_base;
  k.dB = a.dB;
  k.ld_dB = a.ld_dB;
  k.gc_pp = q.pp;
  k.gc_ring = q.ring;
  k.g_ready = reinterpret_cast<uint32_t*>(a.gc_ws);
  k.g_consumed = k.g_ready + q.n_steps * q.pp;
  k.g_unit_done = k.g_consumed + q.n_steps;
  k.g_ring = reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(a.gc_ws) + q.ctr_bytes);
  static int static_smem = -1;
  if (static_smem < 0) {
    cudaFuncAttributes fa;
    INFCL_CUDA_TRY(cudaFuncGetAttributes(&fa, bwd3_kernel<true, false>));
    static_smem = (int)fa.sharedSizeBytes;
  }
  const long long budget = 232448 - ((static_smem + 1023) / 1024) * 1024;
  // producers: resident A (KB x 16 KB) when it leaves >= 4 B-only stages and KB >= 4 (n_stages <= KB), else
  // streamed A (32-KB stages); plus 32 KB of epilogue staging.  Readers: 32-KB stages + 32 KB drain staging.
  const long long stg = 8 * 4096;
  // streamed A by default: with the 32-KB staging, resident A leaves only 4 B stages of 16 KB (64 KB in flight:
  // the producers' MMA waited on TMA 53 % of the time); streamed A keeps 6 stages of 32 KB (192 KB) in flight
  const char* ra = getenv("INFCL_BWD3_RESA");
  const bool resa = ra && atoi(ra) != 0 && k.KB >= 4 && budget - stg - (long long)k.KB * kBoxB >= 4LL * kBoxB;
  const long long stage_bytes = resa ? kBoxB : kWStage3;
  int ns = (int)std::min<long long>(kMaxStages, (budget - stg - (resa ? (long long)k.KB * kBoxB : 0)) / stage_bytes);
  if (resa) ns = std::min(ns, k.KB);
  if (ns < 2) return fail(INFCL_ERR_SHAPE, "3-role backward: smem");
  k.n_stages = ns;
  k.pair_commit = ns % 2 == 0 ? 1 : 0;
  const size_t smem = (size_t)(budget / 1024) * 1024;  // every role takes the whole budget
  k.n_stages_c = std::min((int)((smem - stg) / kStg3), kMaxStages);
  CUtensorMap tmA, tmB, tmG, tmG2, tmGs, tmDT, tmDI;
  infcl_status st;
  if ((st = make_tmap_bf16(&tmA, a.A, a.nrows, a.dk, a.ld, 64, 128))) return st;
  if ((st = make_tmap_bf16(&tmB, a.B, a.ncols, a.dk, a.ld, 64, 128))) return st;
  void* ring = static_cast<uint8_t*>(a.gc_ws) + q.ctr_bytes;
  const uint64_t ring_rows = (uint64_t)q.ring * q.pp * kR3;
  if ((st = make_tmap_bf16(&tmG, ring, ring_rows, kColsPerTile, kColsPerTile, 64, 64))) return st;
  if ((st = make_tmap_bf16(&tmG2, ring, ring_rows, kColsPerTile, kColsPerTile, 64, 128))) return st;
  if ((st = make_tmap_bf16(&tmGs, ring, ring_rows, kColsPerTile, kColsPerTile, 64, 32))) return st;
  if ((st = make_tmap_f32_sw128(&tmDT, a.dB, a.ncols, a.d_out, a.ld_dB, 32, 32))) return st;
  if ((st = make_tmap_f32_sw128(&tmDI, a.dA, a.nrows, a.d_out, a.ld_dA, 32, 32))) return st;
  unsigned long long* dbg = debug_buffer(s);
  k.dbg = dbg;
  auto kern = resa ? (dbg ? bwd3_kernel<true, true> : bwd3_kernel<true, false>)
                   : (dbg ? bwd3_kernel<false, true> : bwd3_kernel<false, false>);
  INFCL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  static int max_clusters = -1;
  if (max_clusters < 0) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(2 * q.npairs);
    cfg.blockDim = dim3(kThreads3);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    INFCL_CUDA_TRY(cudaOccupancyMaxActiveClusters(&max_clusters, (void*)kern, &cfg));
  }
  if (max_clusters < q.npairs)
    return fail(INFCL_ERR_UNSUPPORTED, "3-role backward: only " + std::to_string(max_clusters) +
                                           " CTA pairs co-resident, need " + std::to_string(q.npairs));
  INFCL_CUDA_TRY(cudaMemsetAsync(a.gc_ws, 0, (size_t)q.n_ctr * sizeof(uint32_t), s));
  cudaEvent_t e0 = profile_begin(s);
  kern<<<dim3(2 * q.npairs), dim3(kThreads3), smem, s>>>(tmA, tmB, tmG, tmG2, tmGs, tmDT, tmDI, k);
  INFCL_CUDA_TRY(cudaGetLastError());
  profile_end(1, e0, s);
  ++launch_counter();
  if (dbg) debug_report3(q.pp, q.pc, s);
  return INFCL_OK;
}

}  // namespace infcl
