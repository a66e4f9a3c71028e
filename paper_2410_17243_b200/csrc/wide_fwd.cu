// Wide forward kernel: the forward pass of the fused Inf-CL tile loop (Alg.2 P:258-276 with the symmetric
// column direction) on M=256 CTA-pair tiles.
//
// Why a second forward kernel: the narrow pair kernel (pair_kernel.cu) keeps 128 stationary rows per pair
// resident and issues M=128 pair MMAs (64 tensor cycles each).  Loop-structure probes (probe_walk2_kernel,
// scripts/experiments/walk_probe4.py) show those run at 70-78 % of the tensor rate once the ring handshakes are in the
// loop, while M=256 pair MMAs (128 cycles each) stay at 100 % with the same handshakes.  The forward has no
// TMEM-resident accumulator besides S, so it can afford 256-row pair tiles: S (256 x 256) = A_R * B_C^T with
// tcgen05.mma.cta_group::2 M=256 N=256 (per SM: 128 rows x 256 columns, TMEM lane = row).  At d <= 512 the
// segment's stationary rows are resident (128 rows x d bf16 = up to 128 KB per SM) and each ring stage carries
// one 64-wide K block of B only (16 KB; 5 stages): 32 B/clk of L2->SM operand traffic at the full tensor rate.
// At d = 768 A cannot be resident next to a useful ring, so every 32-KB stage carries one K block of A
// (128 rows) and of B (128 columns) per SM, A coming from L2 after the segment's first tile (64 B/clk, the
// narrow kernel's figure, with 6 stages = 192 KB in flight).
//
// Epilogue: 8 warps; warp (q = warp % 4, u = warp / 4) owns rows 32q..32q+31 (its TMEM lane quarter) and
// columns 128u..128u+127 of the tile, processed as two 64-column chunks with the narrow kernel's per-chunk
// statistics (fwd_chunk_stats, pair_common.cuh).  A chunk's column partials are combined over the 4 row
// quarters through a chunk-parity double-buffered smem exchange and one 128-thread named barrier; each warp
// merges 16 of the chunk's columns into the per-CTA column slot.  Two TMEM S buffers (2 x 256 columns).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "host_utils.h"
#include "kernels.h"
#include "pair_common.cuh"
#include "ptx.cuh"

namespace infcl {

constexpr int kWRows = 256;       // stationary rows per CTA pair (128 per SM)
constexpr int kWStage = 32768;    // ring stage per SM: A block 16 KB + B block 16 KB (one 64-wide K step)
constexpr int kWBufCols = 256;    // TMEM columns per S buffer

template <bool DBG, bool RESA, bool SELF>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    wide_fwd_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ KParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];  // SW128 operands need 1024-B alignment
  if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u)) __trap();
  // RESA (A resident, d <= 512): the segment's 128 stationary rows per SM live in smem (KB x 16-KB K blocks)
  // and the ring stages carry only B (16 KB), halving the L2->SM operand bytes per MMA; the first tile of a
  // segment brings A block kb inside ring stage kb's transaction.  Safe to overwrite: the previous reader of
  // A block kb is the MMA KB ring uses earlier, and the producer's empty wait for this use guarantees every MMA
  // up to n_stages uses earlier has completed (the host keeps n_stages <= KB).
  uint8_t* sA = smem_raw;
  uint8_t* sStage = smem_raw + (RESA ? p.KB * kBoxB : 0);
  constexpr int kStg = RESA ? kBoxB : kWStage;

  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], sfull[2], sfree[2];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float2 xch[2][2][4][64];  // [chunk parity][u][q][column] column partials
  __shared__ float2 rowx[2][128];                     // row partials of the two column halves (segment end)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const Sched S(p.n_rb, p.n_ct, p.npairs, pair);
  const long long nk = S.n_local();

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], 1);
      mbar_init(&sfree[b], 16);  // one arrival per epilogue warp of both CTAs
    }
    fence_mbar_init();
  }
  if (warp == kWarpTMA && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == kWarpMMA) tmem_alloc<2>(&tmem_base, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_base;

  const unsigned long long t_start = DBG ? clock64() : 0ull;
  if (warp == kWarpTMA) {
    // ===================================================================== TMA producer (both CTAs)
    if (lane == 0) {
      WaitClock<DBG> wc(p.dbg, true);
      int stage = 0;
      uint32_t ph = 0;
      long long it = 0;
      while (it < nk) {
        int rb, ct0;
        S.decode(it, rb, ct0);
        const long long seg_end = S.seg_end(it), seg_start = it;
        const int a_row = rb * kWRows + (int)cta * 128;
        for (int ct = ct0; it < seg_end; ++it, ++ct) {  // a segment's column tiles are consecutive
          const int b_row = (ct + (INFCL_MUTATION == 3 && ct == 0 ? 1 : 0)) * kColsPerTile + (int)cta * 128;
          const bool lda = !RESA || it == seg_start;  // this tile's stages bring A blocks
          for (int kb = 0; kb < p.KB; ++kb) {
            ring_acquire(wc, empty, stage, ph, p.pair_commit);
            if (DBG && p.notma) {
              if (cta == 0) mbar_arrive(&full[stage]);
            } else {
              if (cta == 0) mbar_arrive_expect_tx(&full[stage], (lda ? 4 : 2) * kBoxB);
              uint8_t* dst = sStage + stage * kStg;
              if (lda) tma_load_2d_pair(RESA ? sA + kb * kBoxB : dst, &tmA, &full[stage], kb * 64, a_row);
              tma_load_2d_pair(RESA ? dst : dst + kBoxB, &tmB, &full[stage], kb * 64, b_row);
            }
            if (++stage == p.n_stages) {
              stage = 0;
              ph ^= 1;
            }
          }
        }
      }
      wc.flush(0);
    }
  } else if (warp == kWarpMMA) {
    // ===================================================================== MMA issuer (leader CTA)
    if (cta == 0) {
      WaitClock<DBG> wc(p.dbg, lane == 0);
      int stage = 0;
      uint32_t ph = 0, sfph = 0;  // sfph: phase bit of sfree[b] = bit b
      const uint32_t idS = idesc_bf16(256, 256, 0, 0);
      const unsigned long long t_loop = DBG ? clock64() : 0ull;
      for (long long it = 0; it < nk; ++it) {
        const int buf = (int)(it & 1);
        wc.wait(&sfree[buf], ((sfph >> buf) & 1u) ^ 1u, 7, true);
        sfph ^= 1u << buf;
        tc_fence_after();
        const uint32_t dS = tbase + buf * kWBufCols;
        for (int kb = 0; kb < p.KB; ++kb) {
          wc.wait(&full[stage], ph, 5);
          const unsigned long long t_is = DBG ? clock64() : 0ull;
          tc_fence_after();
          const uint32_t st = smem_u32(sStage + stage * kStg);
          const uint32_t sa = RESA ? smem_u32(sA + kb * kBoxB) : st;
          umma_stage_pair<false, 0, 0>(dS, (uint32_t)smem_desc_sw128(sa, 16, 1024),
                                       (uint32_t)smem_desc_sw128(RESA ? st : st + kBoxB, 16, 1024), idS, kb != 0);
          ring_release(empty, stage, p.pair_commit);
          if (DBG) wc.acc[11] += clock64() - t_is;
          if (++stage == p.n_stages) {
            stage = 0;
            ph ^= 1;
          }
        }
        umma_commit_pair_mc_warp(&sfull[buf], 0x3);
      }
      if (DBG) wc.acc[0] += clock64() - t_loop;
      wc.flush(1);
    }
  } else {
    // ===================================================================== epilogue (both CTAs)
    const int q = warp & 3;   // TMEM lane quarter = rows 32q..32q+31 of this CTA's 128
    const int u = warp >> 2;  // column half of the 256-column tile
    const int t0 = lane & 3, t1 = lane >> 2;
    const uint32_t laddr = tbase + ((uint32_t)(q * 32) << 16) + u * 128;
    uint32_t sph = 0;  // phase bit of sfull[b] = bit b
    WaitClock<DBG> wc(p.dbg, lane == 0);
    int cctr = 0;  // chunk counter (xch parity)
    float2* slot = p.col_slots + (long long)blockIdx.x * p.slot_ld;
    long long it = 0;
    while (it < nk) {
      int rb, ct_first;
      S.decode(it, rb, ct_first);
      const long long seg_end = S.seg_end(it);
      const int rowbase = rb * kWRows + (int)cta * 128 + q * 32 + t1;  // launch-local row of v-row 0
      float mrow[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, srow[4] = {0.f, 0.f, 0.f, 0.f};
      const long long seg_start = it;
      for (; it < seg_end; ++it) {
        const int ct = ct_first + (int)(it - seg_start);
        const int buf = (int)(it & 1);
        const bool first_visit = !p.slots_merge && it < p.n_ct;
        wc.wait(&sfull[buf], (sph >> buf) & 1u, 8);
        sph ^= 1u << buf;
        tc_fence_after();
#pragma unroll 1
        for (int ch = 0; ch < 2; ++ch) {
          const int cb = ct * kColsPerTile + u * 128 + ch * 64;  // global column of chunk column 0
          const int cm = cb + q * 16 + lane;                     // the column this lane merges (lanes 0-15)
          float2 pre = make_float2(-INFINITY, 0.f);
          if (!first_visit && lane < 16 && cm < p.ncols) pre = slot[cm];
          const uint32_t lchunk = laddr + buf * kWBufCols + ch * 64;
          float v[64];
          tmem_ld16x256x8(lchunk, v);
          tmem_ld16x256x8(lchunk + (16u << 16), v + 32);
          tmem_ld_wait();
          float4 cs;
          if (DBG && p.noepi) {
            cs = make_float4(-INFINITY, 0.f, -INFINITY, 0.f);
          } else {
            cs = fwd_chunk_stats<SELF>(v, lchunk, rowbase, cb, p, lane, mrow, srow);
          }
          if (ch == 1) {  // release this S buffer (per warp) after the last TMEM read of the tile
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&sfree[buf], 0);
          }
          // xch is double-buffered by chunk parity: a warp rewrites buffer c&1 at chunk c+2 only after passing
          // chunk c+1's barrier, i.e. after all four warps finished reading chunk c
          float2(*xb)[4][64] = xch[cctr & 1];
          *reinterpret_cast<float4*>(&xb[u][q][2 * lane]) = cs;
          named_bar_sync(2 + u, 128);
          {  // lanes 0-15 merge row quarters 0,1 and lanes 16-31 quarters 2,3 of column q*16 + (lane & 15)
            const int c = q * 16 + (lane & 15), hq = lane >> 4;
            float2 a = merge2(xb[u][2 * hq][c], xb[u][2 * hq + 1][c]);
            float2 o;
            o.x = __shfl_xor_sync(0xffffffffu, a.x, 16);
            o.y = __shfl_xor_sync(0xffffffffu, a.y, 16);
            a = merge2(a, o);
            if (lane < 16) {
              if (!first_visit) a = merge2(pre, a);
              if (cm < p.ncols) slot[cm] = a;
            }
          }
          ++cctr;
        }
      }
      // segment end: merge each row's 4 lane slices (t0), then its 2 column halves (u); write the row partial
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
        if (t0 == 0) rowx[u][q * 32 + 16 * (ri >> 1) + 8 * (ri & 1) + t1] = a;
      }
      named_bar_sync(1, 256);
      if (u == 0) {
        const int r = q * 32 + lane;
        if (rb * kWRows + (int)cta * 128 + r < p.nrows)
          p.row_parts[S.seg_slot(rb) * kWRows + cta * 128 + r] = merge2(rowx[0][r], rowx[1][r]);
      }
      named_bar_sync(1, 256);
    }
    wc.flush(2 + (warp & 1));
  }
  __syncwarp();
  if (DBG && p.dbg && threadIdx.x == 0) atomicAdd(p.dbg + 4 * 16 + 15, (unsigned long long)(clock64() - t_start));
  tc_fence_before();
  cluster_sync();
  if (warp == kWarpMMA) tmem_dealloc<2>(tbase, 512);
}

// ------------------------------------------------------------------------------------------ host side
bool wide_forward_enabled() {
  const char* e = getenv("INFCL_FWD_NARROW");  // A/B diagnostic and test switch: the narrow forward kernel
  return !(e && *e && *e != '0');
}

PassGeom wide_geom(int nrows, int ncols) {
  PassGeom g;
  g.rpp = kWRows;
  g.n_rb = (nrows + kWRows - 1) / kWRows;
  g.n_ct = (ncols + kColsPerTile - 1) / kColsPerTile;
  g.n_items = (long long)g.n_rb * g.n_ct;
  const int pairs = max_pairs();
  g.npairs = (int)std::min<long long>(pairs, g.n_items);
  return g;
}

infcl_status launch_wide_forward(const PassArgs& a, cudaStream_t s) {
  if (a.dk > kMaxD) return fail(INFCL_ERR_SHAPE, "feature dim above kernel limit 768");
  const PassGeom g = wide_geom(a.nrows, a.ncols);
  KParams k{};
  k.nrows = a.nrows;
  k.ncols = a.ncols;
  k.dk = a.dk;
  k.KB = (a.dk + 63) / 64;
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
  unsigned long long* dbg = debug_buffer(s);
  k.dbg = dbg;
  static int static_smem = -1;
  if (static_smem < 0) {
    cudaFuncAttributes fa;
    INFCL_CUDA_TRY(cudaFuncGetAttributes(&fa, wide_fwd_kernel<false, false, false>));
    static_smem = (int)fa.sharedSizeBytes;
  }
  const long long budget = 232448 - ((static_smem + 1023) / 1024) * 1024;
  // A resident when it leaves >= 4 B-only stages (KB <= 8, i.e. d <= 512) and KB >= 4; n_stages <= KB keeps
  // the A-block overwrite safe (see the kernel).  INFCL_FWD_STREAM_A=1: A/B switch back to streamed A.
  const char* sa_env = getenv("INFCL_FWD_STREAM_A");
  const bool resa = !(sa_env && *sa_env && *sa_env != '0') && k.KB >= 4 &&
                    budget - (long long)k.KB * kBoxB >= 4LL * kBoxB;
  const long long stage_bytes = resa ? kBoxB : kWStage;
  int ns = (int)std::min<long long>(kMaxStages, (budget - (resa ? (long long)k.KB * kBoxB : 0)) / stage_bytes);
  if (resa) ns = std::min(ns, k.KB);
  if (const char* e = getenv("INFCL_STAGES")) ns = std::max(2, std::min(ns, atoi(e)));
  k.n_stages = ns;
  k.pair_commit = (ns % 2 == 0 && !getenv("INFCL_NO_PAIR_COMMIT")) ? 1 : 0;
  const size_t smem = (size_t)ns * stage_bytes + (resa ? (size_t)k.KB * kBoxB : 0);
  CUtensorMap tmA, tmB;
  infcl_status st = make_tmap_bf16(&tmA, a.A, a.nrows, a.dk, a.ld, 64, 128);
  if (st) return st;
  if ((st = make_tmap_bf16(&tmB, a.B, a.ncols, a.dk, a.ld, 64, 128))) return st;
  k.noepi = getenv("INFCL_DEBUG_NOEPI") != nullptr;
  k.notma = getenv("INFCL_DEBUG_NOTMA") != nullptr;
  // self-masked (NT-Xent) launches use their own instantiation: the self mask in the CLIP kernel's epilogue cost
  // register spills and 17 % forward time (round-2 bench)
  auto kern = a.self_mask ? (resa ? wide_fwd_kernel<false, true, true> : wide_fwd_kernel<false, false, true>)
              : resa ? (dbg ? wide_fwd_kernel<true, true, false> : wide_fwd_kernel<false, true, false>)
                     : (dbg ? wide_fwd_kernel<true, false, false> : wide_fwd_kernel<false, false, false>);
  INFCL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0 = profile_begin(s);
  kern<<<dim3(2 * g.npairs), dim3(kThreads), smem, s>>>(tmA, tmB, k);
  INFCL_CUDA_TRY(cudaGetLastError());
  profile_end(0, e0, s);
  if (dbg) debug_report("FWD(wide)", g.npairs, s);
  ++launch_counter();
  return INFCL_OK;
}

}  // namespace infcl
