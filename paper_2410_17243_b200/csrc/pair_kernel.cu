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
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM alloc + MMA issuer (leader CTA), warps 2-5
// epilogue (TMEM lane quarter = warp % 4).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <utility>
#include <vector>

#include "host_utils.h"
#include "kernels.h"
#include "ptx.cuh"

namespace infcl {

// ---- optional per-launch event timing (infcl_profile_*)
struct ProfState {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[2];
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

constexpr int kThreads = 192;
constexpr int kBox = 8192;     // one TMA box: 64 rows x 64 bf16 (128 B, SW128)
constexpr int kStage = 16384;  // one ring stage: two boxes
constexpr int kMaxStages = 12;
constexpr int kSmemBudget = 232448 - 8192;  // 227 KB opt-in minus static smem and slack

struct KParams {
  int nrows, ncols, dk, KB, NDC;
  int n_rb, n_ct, npairs, n_stages;
  long long n_items;
  float k2, scale;
  int diag_on;
  float2* col_slots;
  long long slot_ld;
  float2* row_parts;
  float* diag_out;
  const float* lse_row2;
  const float* lse_col2;
  float* dA;
  int ld_dA, d_out;
  const float* grad;
  float coef_base;
};

__device__ __forceinline__ long long item_begin(long long n_items, int npairs, int p) {
  return (long long)p * n_items / npairs;
}

__device__ __forceinline__ float2 merge2(float2 a, float2 b) {
  const float M = fmaxf(a.x, b.x);
  if (M == -INFINITY) return make_float2(-INFINITY, 0.f);
  return make_float2(M, a.y * ex2(a.x - M) + b.y * ex2(b.x - M));
}

// Transposed butterfly reduction of 32 values per lane: afterwards lane l holds op over the 32 lanes of
// the value originally at index l (5 rounds, 31 shuffles).
template <bool IS_MAX>
__device__ __forceinline__ float xreduce32(float (&t)[32], int lane) {
#define XR_ROUND(O, N)                                                 \
  {                                                                    \
    const bool up = (lane & (O)) != 0;                                 \
    _Pragma("unroll") for (int i = 0; i < (N); ++i) {                  \
      const float send = up ? t[i] : t[i + (N)];                       \
      const float keep = up ? t[i + (N)] : t[i];                       \
      const float recv = __shfl_xor_sync(0xffffffffu, send, (O));      \
      t[i] = IS_MAX ? fmaxf(keep, recv) : keep + recv;                 \
    }                                                                  \
  }
  XR_ROUND(16, 16)
  XR_ROUND(8, 8)
  XR_ROUND(4, 4)
  XR_ROUND(2, 2)
  XR_ROUND(1, 1)
#undef XR_ROUND
  return t[0];
}

template <bool BWD>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ KParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sG = sA + p.KB * kBox;
  uint8_t* sStage = sG + (BWD ? 4 * kBox : 0);

  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ __align__(8) uint64_t afull, afree, sfull[2], sfree[2], gready, gfree, dafull, dafree;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float cmx[2][2][128];
  __shared__ __align__(16) float csm[2][2][128];
  __shared__ float2 rowx[64];
  __shared__ __align__(16) float cval[2][256];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const long long it0 = item_begin(p.n_items, p.npairs, pair);
  const long long it1 = item_begin(p.n_items, p.npairs, pair + 1);
  constexpr uint32_t kTmemCols = BWD ? 512 : 256;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&afull, 1);
    mbar_init(&afree, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], 1);
      mbar_init(&sfree[b], 2);
    }
    mbar_init(&gready, 2);
    mbar_init(&gfree, 1);
    mbar_init(&dafull, 1);
    mbar_init(&dafree, 2);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc<2>(&tmem_base, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_base;

  if (warp == 0) {
    // ===================================================================== TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0, aph = 0;
      auto load_stage = [&](int c0a, int c1a, int c0b, int c1b) {
        mbar_wait(&empty[stage], ph ^ 1, 1);
        if (cta == 0) mbar_arrive_expect_tx(&full[stage], 2 * kStage);
        uint8_t* dst = sStage + stage * kStage;
        tma_load_2d_pair(dst, &tmB, &full[stage], c0a, c1a);
        tma_load_2d_pair(dst + kBox, &tmB, &full[stage], c0b, c1b);
        if (++stage == p.n_stages) {
          stage = 0;
          ph ^= 1;
        }
      };
      auto load_S = [&](int ct) {
        const int j0 = ct * kColsPerTile + (int)cta * 128;
        for (int kb = 0; kb < p.KB; ++kb) load_stage(kb * 64, j0, kb * 64, j0 + 64);
      };
      auto load_dA = [&](int ct) {
        for (int tc = 0; tc < p.NDC; ++tc) {
          const int d0 = tc * 256 + (int)cta * 128;
          for (int jc = 0; jc < 4; ++jc) load_stage(d0, ct * kColsPerTile + jc * 64, d0 + 64, ct * kColsPerTile + jc * 64);
        }
      };
      long long it = it0;
      while (it < it1) {
        const int rb = (int)(it / p.n_ct);
        const long long seg_end = std::min<long long>(it1, (long long)(rb + 1) * p.n_ct);
        mbar_wait(&afree, aph ^ 1, 2);
        aph ^= 1;
        if (cta == 0) mbar_arrive_expect_tx(&afull, 2u * p.KB * kBox);
        for (int kb = 0; kb < p.KB; ++kb)
          tma_load_2d_pair(sA + kb * kBox, &tmA, &afull, kb * 64, rb * kRowsPerPair + (int)cta * 64);
        int prev = -1;
        for (; it < seg_end; ++it) {
          const int ct = (int)(it % p.n_ct);
          load_S(ct);
          if (BWD && prev >= 0) load_dA(prev);
          prev = ct;
        }
        if (BWD) load_dA(prev);
      }
    }
  } else if (warp == 1) {
    // ===================================================================== MMA issuer (leader CTA)
    if (cta == 0 && lane == 0) {
      int stage = 0;
      uint32_t ph = 0, aph = 0, gph = 0, dph = 0;
      uint32_t sfph[2] = {0, 0};
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
          mbar_wait_cluster(&dafree, dph ^ 1, 3);
          dph ^= 1;
        }
        mbar_wait_cluster(&gready, gph, 4);
        gph ^= 1;
        tc_fence_after();
        for (int tc = 0; tc < p.NDC; ++tc) {
          for (int jc = 0; jc < 4; ++jc) {
            mbar_wait(&full[stage], ph, 5);
            tc_fence_after();
            const uint32_t sa = smem_u32(sStage + stage * kStage);
            const uint32_t sb = smem_u32(sG + jc * kBox);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = smem_desc_sw128(sa + k * 2048, kBox, 1024);  // MN-major B_C^T
              const uint64_t bd = smem_desc_sw128(sb + k * 32, 16, 1024);      // K-major G
              umma_bf16<2>(tbase + 128 + tc * 128, ad, bd, idD, (first && jc == 0 && k == 0) ? 0u : 1u);
            }
            umma_commit_pair_mc(&empty[stage], 0x3);
            advance();
          }
        }
        umma_commit_pair_mc(&gfree, 0x3);
      };
      long long it = it0;
      while (it < it1) {
        const int rb = (int)(it / p.n_ct);
        const long long seg_end = std::min<long long>(it1, (long long)(rb + 1) * p.n_ct);
        mbar_wait_cluster(&afull, aph, 6);
        aph ^= 1;
        tc_fence_after();
        bool have_prev = false, first_dA = true;
        for (; it < seg_end; ++it) {
          const int buf = BWD ? 0 : (tile_ctr & 1);
          mbar_wait_cluster(&sfree[buf], sfph[buf] ^ 1, 7);
          sfph[buf] ^= 1;
          tc_fence_after();
          const uint32_t dS = tbase + buf * 128;
          for (int kb = 0; kb < p.KB; ++kb) {
            mbar_wait(&full[stage], ph, 5);
            tc_fence_after();
            const uint32_t sa = smem_u32(sA + kb * kBox);
            const uint32_t sb = smem_u32(sStage + stage * kStage);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              umma_bf16<2>(dS, smem_desc_sw128(sa + k * 32, 16, 1024), smem_desc_sw128(sb + k * 32, 16, 1024), idS,
                           (kb | k) != 0);
            }
            umma_commit_pair_mc(&empty[stage], 0x3);
            advance();
          }
          umma_commit_pair_mc(&sfull[buf], 0x3);
          if (it + 1 == seg_end) umma_commit_pair_mc(&afree, 0x3);
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
          umma_commit_pair_mc(&dafull, 0x3);
        }
      }
    }
  } else {
    // ===================================================================== epilogue (both CTAs)
    const int q = warp & 3;        // TMEM lane quarter
    const int h = q >> 1;          // column half of the 256-column tile
    const int rh = q & 1;          // which 32 of the CTA's 64 rows
    const int r = rh * 32 + lane;  // row within this CTA's 64
    const int et = threadIdx.x - 64;
    const uint32_t laddr = tbase + ((uint32_t)(q * 32) << 16);
    uint32_t sph[2] = {0, 0}, gfph = 0, daph = 0;
    int tile_ctr = 0;
    const float k2 = p.k2;
    float coef = 0.f;
    if (BWD) coef = p.coef_base * __ldg(p.grad);
    long long it = it0;
    while (it < it1) {
      const int rb = (int)(it / p.n_ct);
      const long long seg_end = std::min<long long>(it1, (long long)(rb + 1) * p.n_ct);
      const int ig = rb * kRowsPerPair + (int)cta * 64 + r;
      const bool row_ok = ig < p.nrows;
      float m = -INFINITY, sig = 0.f;
      float r2 = 0.f;
      if (BWD && row_ok) r2 = __ldg(p.lse_row2 + ig);
      for (; it < seg_end; ++it) {
        const int ct = (int)(it % p.n_ct);
        const int buf = BWD ? 0 : (tile_ctr & 1);
        const int cbase = ct * kColsPerTile + h * 128;  // global column of this thread's local column 0
        float* cv = cval[tile_ctr & 1];
        if (BWD) {
          const int j0 = ct * kColsPerTile + et * 2;
          cv[et * 2] = j0 < p.ncols ? __ldg(p.lse_col2 + j0) : 0.f;
          cv[et * 2 + 1] = j0 + 1 < p.ncols ? __ldg(p.lse_col2 + j0 + 1) : 0.f;
        }
        mbar_wait(&sfull[buf], sph[buf], 8);
        sph[buf] ^= 1;
        tc_fence_after();
        float v[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(laddr + buf * 128 + c * 32, v + c * 32);
        tmem_ld_wait();
        tc_fence_before();
        named_bar_sync(1, 128);
        if (et == 0) mbar_arrive_cluster(&sfree[buf], 0);
        const bool diag_tile = p.diag_on && ig >= cbase && ig < cbase + 128;

        if constexpr (!BWD) {
          // ---------------------------------------------------------- forward statistics
          if (diag_tile && row_ok && p.diag_out) {
            float dv = 0.f;
#pragma unroll
            for (int j = 0; j < 128; ++j) dv = (cbase + j == ig) ? v[j] : dv;
            p.diag_out[ig] = dv * p.scale;
          }
          float mt = -INFINITY;
#pragma unroll
          for (int j = 0; j < 128; ++j) {
            const bool ok = row_ok && (cbase + j < p.ncols);
            v[j] = ok ? v[j] * k2 : -INFINITY;
            mt = fmaxf(mt, v[j]);
          }
          const float mn = fmaxf(m, mt);
          if (mn != -INFINITY) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < 128; ++j) acc += ex2(v[j] - mn);
            sig = sig * ex2(m - mn) + acc;
            m = mn;
          }
          // column max over this warp's 32 rows -> lane l holds column 32c + l
          float cmax[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float t[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) t[i] = v[c * 32 + i];
            cmax[c] = xreduce32<true>(t, lane);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) cmx[h][rh][c * 32 + lane] = cmax[c];
          named_bar_sync(2 + h, 64);
          float csum[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float t[32];
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 a = *reinterpret_cast<const float4*>(&cmx[h][0][c * 32 + i]);
              const float4 b = *reinterpret_cast<const float4*>(&cmx[h][1][c * 32 + i]);
              const float M0 = fmaxf(a.x, b.x), M1 = fmaxf(a.y, b.y), M2 = fmaxf(a.z, b.z), M3 = fmaxf(a.w, b.w);
              t[i + 0] = M0 == -INFINITY ? 0.f : ex2(v[c * 32 + i + 0] - M0);
              t[i + 1] = M1 == -INFINITY ? 0.f : ex2(v[c * 32 + i + 1] - M1);
              t[i + 2] = M2 == -INFINITY ? 0.f : ex2(v[c * 32 + i + 2] - M2);
              t[i + 3] = M3 == -INFINITY ? 0.f : ex2(v[c * 32 + i + 3] - M3);
            }
            csum[c] = xreduce32<false>(t, lane);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) csm[h][rh][c * 32 + lane] = csum[c];
          named_bar_sync(2 + h, 64);
          if (rh == 0) {
            const bool first_visit = (it - it0) < p.n_ct;
            float2* slot = p.col_slots + (long long)blockIdx.x * p.slot_ld;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int jl = c * 32 + lane;
              const int jg = cbase + jl;
              if (jg < p.ncols) {
                float2 nw = make_float2(fmaxf(cmx[h][0][jl], cmx[h][1][jl]), csm[h][0][jl] + csm[h][1][jl]);
                if (!first_visit) nw = merge2(slot[jg], nw);
                slot[jg] = nw;
              }
            }
          }
        } else {
          // ---------------------------------------------------------- backward: G tile -> smem
          const float* cvh = cv + h * 128;
          uint32_t pk[64];
#pragma unroll
          for (int j = 0; j < 128; j += 4) {
            const float4 c4 = *reinterpret_cast<const float4*>(cvh + j);
            float g[4];
            const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int jg = cbase + j + u;
              const float y = v[j + u] * k2;
              const bool ok = row_ok && jg < p.ncols && !(p.diag_on && jg == ig);
              g[u] = ok ? ex2(y - r2) + ex2(y - cc[u]) : 0.f;
            }
            pk[j / 2] = pack_bf16(g[0], g[1]);
            pk[j / 2 + 1] = pack_bf16(g[2], g[3]);
          }
          mbar_wait(&gfree, gfph ^ 1, 9);
          gfph ^= 1;
          const uint32_t gb = smem_u32(sG) + (2 * h) * kBox + r * 128;
#pragma unroll
          for (int kb = 0; kb < 2; ++kb)
#pragma unroll
            for (int c16 = 0; c16 < 8; ++c16)
              st_shared_v4(gb + kb * kBox + ((c16 ^ (r & 7)) << 4), pk[kb * 32 + c16 * 4 + 0], pk[kb * 32 + c16 * 4 + 1],
                           pk[kb * 32 + c16 * 4 + 2], pk[kb * 32 + c16 * 4 + 3]);
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (et == 0) mbar_arrive_cluster(&gready, 0);
        }
        ++tile_ctr;
      }
      if constexpr (!BWD) {
        // merge the two column halves of each row, write this segment's row partial
        if (h == 1) rowx[r] = make_float2(m, sig);
        named_bar_sync(1, 128);
        if (h == 0 && row_ok)
          p.row_parts[(long long)(pair + rb) * kRowsPerPair + cta * 64 + r] = merge2(make_float2(m, sig), rowx[r]);
      } else {
        // drain dA^T (128 d-rows of each 256-chunk x 128 pair rows) with red.add into dA
        mbar_wait(&dafull, daph, 10);
        daph ^= 1;
        tc_fence_after();
        for (int tc = 0; tc < p.NDC; ++tc) {
          const int d = tc * 256 + (int)cta * 128 + q * 32 + lane;
          const int row0 = rb * kRowsPerPair;
          for (int c = 0; c < 4; ++c) {
            float v[32];
            tmem_ld32(laddr + 128 + tc * 128 + c * 32, v);
            tmem_ld_wait();
            if (d < p.d_out) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (row0 + c * 32 + i < p.nrows)
                  red_add_f32(p.dA + (long long)(row0 + c * 32 + i) * p.ld_dA + d, coef * v[i]);
            }
          }
        }
        tc_fence_before();
        named_bar_sync(1, 128);
        if (et == 0) mbar_arrive_cluster(&dafree, 0);
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) tmem_dealloc<2>(tbase, kTmemCols);
}

// ------------------------------------------------------------------------------------------ host side
PassGeom pass_geom(int nrows, int ncols) {
  PassGeom g;
  g.n_rb = (nrows + kRowsPerPair - 1) / kRowsPerPair;
  g.n_ct = (ncols + kColsPerTile - 1) / kColsPerTile;
  g.n_items = (long long)g.n_rb * g.n_ct;
  int pairs = std::max(1, num_sms() / 2);
  g.npairs = (int)std::min<long long>(pairs, g.n_items);
  return g;
}

template <bool BWD>
static infcl_status launch_pair(const PassArgs& a, cudaStream_t s) {
  if (a.dk > kMaxD) return fail(INFCL_ERR_SHAPE, "feature dim above kernel limit 768");
  const PassGeom g = pass_geom(a.nrows, a.ncols);
  KParams k{};
  k.nrows = a.nrows;
  k.ncols = a.ncols;
  k.dk = a.dk;
  k.KB = (a.dk + 63) / 64;
  k.NDC = (a.dk + 255) / 256;
  k.n_rb = g.n_rb;
  k.n_ct = g.n_ct;
  k.npairs = g.npairs;
  k.n_items = g.n_items;
  k.k2 = a.scale * 1.4426950408889634f;
  k.scale = a.scale;
  k.diag_on = a.diag_on;
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
  const size_t fixed = 1024 + (size_t)k.KB * kBox + (BWD ? 4 * kBox : 0);
  int ns = (int)((kSmemBudget - (long long)fixed) / kStage);
  ns = std::min(ns, kMaxStages);
  if (ns < 2) return fail(INFCL_ERR_SHAPE, "feature dim too large for the smem budget");
  k.n_stages = ns;
  const size_t smem = fixed + (size_t)ns * kStage;

  CUtensorMap tmA, tmB;
  infcl_status st = make_tmap_bf16(&tmA, a.A, a.nrows, a.dk, a.ld, 64, 64);
  if (st) return st;
  if ((st = make_tmap_bf16(&tmB, a.B, a.ncols, a.dk, a.ld, 64, 64))) return st;

  auto kern = pair_kernel<BWD>;
  INFCL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof().on) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  kern<<<dim3(2 * g.npairs), dim3(kThreads), smem, s>>>(tmA, tmB, k);
  INFCL_CUDA_TRY(cudaGetLastError());
  if (prof().on) {
    cudaEventRecord(e1, s);
    prof().ev[BWD ? 1 : 0].push_back({e0, e1});
  }
  ++launch_counter();
  return INFCL_OK;
}

infcl_status launch_pair_forward(const PassArgs& a, cudaStream_t s) { return launch_pair<false>(a, s); }

void profile_enable(bool on) {
  prof_clear();
  prof().on = on;
}

infcl_status profile_read(int kind, int* launches, double* total_ms) {
  if (kind < 0 || kind > 1 || !launches || !total_ms) return fail(INFCL_ERR_INVALID_ARG, "bad profile query");
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
infcl_status launch_pair_backward(const PassArgs& a, cudaStream_t s) { return launch_pair<true>(a, s); }

}  // namespace infcl
