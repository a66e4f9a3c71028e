// Pieces shared by the pair kernels (pair_kernel.cu: narrow forward + backward; wide_fwd.cu: wide forward):
// launch constants, kernel parameters, the column-synchronous schedule, debug wait timers, and the forward
// epilogue's per-chunk statistics (Eq.4/Eq.5 tile pieces for rows and columns).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "kernels.h"
#include "ptx.cuh"

namespace infcl {

constexpr int kThreads = 320;  // warps 0-7 epilogue, warp 8 TMA, warp 9 MMA
constexpr int kWarpTMA = 8, kWarpMMA = 9;
constexpr int kThreadsGC = 352;  // fused backward: + warp 10, the producers' G ring signal warp
constexpr int kWarpSignal = 10;
constexpr int kBox = 8192;     // A_R / G block: 64 rows x 64 bf16 (128 B, SW128)
constexpr int kBoxB = 16384;   // streamed B box: 128 rows x 64 bf16 (128 B, SW128)
constexpr int kMaxStages = 16;

struct KParams {
  int nrows, ncols, dk, KB, KC, NDC;
  int n_rb, n_ct, npairs, n_stages;
  int sbox, stage_bytes;  // B boxes per ring stage (forward 1 = 16 KB stages, backward 2 = 32 KB) and its bytes
  long long n_items;
  float k2, scale;
  int diag_on, row_off, slots_merge;
  int self_mask;  // column i + row_off of row i is the row's own view: excluded (-inf / G = 0), NT-Xent self-similarity
  int pair_commit;  // even ring: one tcgen05.commit per two stages (empty[even] releases the pair)
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
  float* tail_scratch;      // backward: per-pair partials of split tail row blocks (deterministic) or nullptr
  // fused backward (GC): pairs [0, gc_pp) produce (S, G, dA; G tiles -> global ring), pairs [gc_pp, npairs)
  // consume the ring (dB^T += A^T G per column tile over each wave of gc_pp row blocks)
  int gc_pp, gc_ring, n_stages_c;
  int gc_hint;  // L2 policies (INFCL_GC_HINT bits): 1 consumer G loads evict_first, 2 producer G stores evict_last,
                // 4 consumer A loads evict_last
  uint16_t* g_ring;      // [gc_ring * gc_pp * 128][256] bf16 G tiles (row-major; TMA view: tmG)
  uint32_t* g_ready;     // [n_steps] producer CTAs (2 per pair) whose rows of step g's tiles are in the ring
  uint32_t* g_consumed;  // [n_steps] consumers (nparts) that have read step g's ring slot
  uint32_t* g_unit_done; // [n_ct * nparts] drain warps (16 per wave) whose reductions of the unit are complete
  float* dB;             // dB (dT) accumulated with red.add (column side)
  int ld_dB;
  unsigned long long* dbg;  // optional per-tag wait-cycle accumulators (INFCL_DEBUG_WAITS)
  int noepi;                // diagnostic: epilogue skips its math (results invalid; INFCL_DEBUG_NOEPI)
  int notma;                // diagnostic: producer signals stages without loading (results invalid)
};

// Column-synchronous schedule.  Full waves: pair p owns row block w*P + p for w < W = n_rb / P and sweeps all
// column tiles in order, so all pairs stream the same B tiles at about the same time (each tile is read from
// HBM once and served from L2 to the other pairs).  Tail: the remaining R = n_rb - W*P row blocks x n_ct tiles
// are split into P contiguous ranges (row-major), so the last wave stays balanced.  Segment = consecutive
// items of one row block; row-partial slot of a segment: rb (full waves) or n_rb + p + (rb - W*P) (tail).
// whole_tail (fused backward): tail row block W*P + p goes whole to pair p (no row block is split, so every G
// tile of the last wave has exactly one producer and every dA row block one drain).
struct Sched {
  int P, W, n_ct, n_rb, pair;
  long long tb, te;  // this pair's tail range (tail item indices)
  __device__ Sched(int n_rb_, int n_ct_, int P_, int pair_, bool whole_tail = false)
      : P(P_), n_ct(n_ct_), n_rb(n_rb_), pair(pair_) {
    W = n_rb / P;
    const int R = n_rb - W * P;
    const long long T = (long long)R * n_ct;
    if (whole_tail) {
      tb = pair < R ? (long long)pair * n_ct : T;
      te = pair < R ? tb + n_ct : T;
    } else {
      tb = (long long)pair * T / P;
      te = (long long)(pair + 1) * T / P;
    }
  }
  __device__ long long n_local() const { return (long long)W * n_ct + (te - tb); }
  __device__ void decode(long long k, int& rb, int& ct) const {
    const long long kw = (long long)W * n_ct;
    if (k < kw) {
      rb = (int)(k / n_ct) * P + pair;
      ct = (int)(k % n_ct);
    } else {
      const long long t = tb + (k - kw);
      rb = W * P + (int)(t / n_ct);
      ct = (int)(t % n_ct);
    }
  }
  __device__ long long seg_end(long long k) const {  // exclusive local index where k's segment ends
    const long long kw = (long long)W * n_ct;
    if (k < kw) return (k / n_ct + 1) * n_ct;
    const long long t = tb + (k - kw);
    return kw + std::min<long long>(te, (t / n_ct + 1) * n_ct) - tb;
  }
  __device__ long long seg_slot(int rb) const { return rb < W * P ? rb : (long long)n_rb + pair + (rb - W * P); }
};

// spin until a global counter (written by other CTAs with release semantics) reaches v; watchdog as mbar_wait
__device__ __forceinline__ void spin_geq(const uint32_t* ctr, uint32_t v, int tag) {
  if (ld_acquire_gpu(ctr) >= v) return;
  const unsigned long long t0 = clock64();
  while (ld_acquire_gpu(ctr) < v) {
    __nanosleep(32);
    if (clock64() - t0 > INFCL_WATCHDOG_CYCLES) watchdog_fire(tag, v);
  }
}

__device__ __forceinline__ float2 merge2(float2 a, float2 b) {
  const float M = fmaxf(a.x, b.x);
  if (M == -INFINITY) return make_float2(-INFINITY, 0.f);
  return make_float2(M, a.y * ex2(a.x - M) + b.y * ex2(b.x - M));
}

template <bool ON>
struct WaitClock {
  // every lane of the role times its waits (a lane-dependent branch here would diverge a converged warp and
  // hide the wait of the lanes that did not time); only lane 0 flushes
  unsigned long long* dbg;
  bool leader;
  unsigned long long acc[ON ? 12 : 1];
  __device__ WaitClock(unsigned long long* d, bool lead) : dbg(d), leader(lead) {
#pragma unroll
    for (int i = 0; i < (ON ? 12 : 1); ++i) acc[i] = 0;
  }
  __device__ __forceinline__ void wait(uint64_t* bar, uint32_t par, int tag, bool cluster = false) {
    if (!ON || !dbg) {
      if (cluster) mbar_wait_cluster(bar, par, tag);
      else mbar_wait(bar, par, tag);
      return;
    }
    const unsigned long long t0 = clock64();
    if (cluster) mbar_wait_cluster(bar, par, tag);
    else mbar_wait(bar, par, tag);
    acc[tag] += clock64() - t0;
  }
  __device__ void flush(int role) {
    if constexpr (ON) {
      if (!dbg || !leader) return;
      for (int i = 0; i < 12; ++i)
        if (acc[i]) atomicAdd(dbg + role * 16 + i, acc[i]);
    }
  }
};


// Ring stage release / acquire with optional pairing: a commit costs the tensor pipe a bubble, so with an even
// number of stages the MMA warp commits once per two stages (to empty[s-1] after odd stage s; the commit fires
// when all prior MMAs complete, i.e. it covers both) and the producer waits only before even stages.
// (scripts/experiments/walk_probe5.py: -6 % cycles per MMA in the loop-structure probe.)
__device__ __forceinline__ void ring_release(uint64_t* empty, int stage, int pair_commit) {
  if (!pair_commit) umma_commit_pair_mc_warp(&empty[stage], 0x3);
  else if (stage & 1) umma_commit_pair_mc_warp(&empty[stage - 1], 0x3);
}
template <bool DBG>
__device__ __forceinline__ void ring_acquire(WaitClock<DBG>& wc, uint64_t* empty, int stage, uint32_t ph,
                                             int pair_commit) {
  if (!pair_commit || !(stage & 1)) wc.wait(&empty[stage], ph ^ 1, 1);
}

// Forward statistics of one 64-column chunk of an S tile held by this warp in the tcgen05.ld 16x256b layout:
// t0 = lane & 3, t1 = lane >> 2; value v[eta*32 + rho*4 + kap*2 + c] is row rowbase + 16*eta + 8*kap (launch-
// local row index; rowbase already includes t1), column cb + 8*rho + 2*t0 + c.  `lchunk` = TMEM address of the
// chunk (lanes +16 for eta = 1), re-read only by the exact fallback.  Row references are thread-local maxima
// (any upper bound works for shared exponentials), so rows need no shuffles; column sums reduce 4 rows
// in-thread, then 8 lanes (3 butterfly rounds).  Updates the running (mrow, srow) of the thread's 4 rows
// (base-2 units), writes x_ii for diagonal rows, and returns (m0, S0, m1, S1): the (max, sum) partial of
// columns cb + 2*lane and cb + 2*lane + 1 over the warp's 32 rows.
// INFCL_FWD_POLY = k (A/B builds only): the row exponentials of the first k of every 8 column pairs are computed
// on the FMA pipe instead of MUFU (Cody-Waite split + degree-4 polynomial, packed f32x2), Eq.5's exp
#ifndef INFCL_FWD_POLY
#define INFCL_FWD_POLY 0
#endif
// INFCL_FWD_FMAX3 = 1 (A/B builds only): the row maxima through 3-input FMNMX3 trees (measured 2 % slower)
#ifndef INFCL_FWD_FMAX3
#define INFCL_FWD_FMAX3 0
#endif
// 2^t for t <= 0 (t = -inf -> 0): t = n + f, n = round(t) by the 1.5 * 2^23 shifter, f in [-0.5, 0.5];
// 2^f by a degree-4 minimax polynomial (max relative error 3.7e-6, below bf16 / the 2e-3 LSE gate), then n is
// added to the exponent field
__device__ __forceinline__ float2 ex2_poly2(float2 t) {
  const float2 lo = make_float2(-126.f, -126.f);
  t = make_float2(fmaxf(t.x, lo.x), fmaxf(t.y, lo.y));  // -inf and deep underflow -> 2^-126 (negligible)
  const float2 sh = make_float2(12582912.f, 12582912.f);
  const float2 j = __fadd2_rn(t, sh);
  const float2 f = __fadd2_rn(t, __ffma2_rn(j, make_float2(-1.f, -1.f), sh));  // t - (j - sh) = t - n
  float2 q = __ffma2_rn(f, make_float2(1.3333558e-3f, 1.3333558e-3f), make_float2(9.6181291e-3f, 9.6181291e-3f));
  q = __ffma2_rn(q, f, make_float2(5.5504109e-2f, 5.5504109e-2f));
  q = __ffma2_rn(q, f, make_float2(2.4022652e-1f, 2.4022652e-1f));
  q = __ffma2_rn(q, f, make_float2(6.9314718e-1f, 6.9314718e-1f));
  q = __ffma2_rn(q, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(j.y) << 23)));
}

// SELF: the launch may be self-masked (NT-Xent); a separate instantiation, so the CLIP kernels carry none of it.
template <bool SELF>
__device__ __forceinline__ float4 fwd_chunk_stats(float (&v)[64], uint32_t lchunk, int rowbase, int cb,
                                                  const KParams& p, int lane, float (&mrow)[4], float (&srow)[4]) {
  const float k2 = p.k2;
  const int t0 = lane & 3;
  bool rok[4];
#pragma unroll
  for (int ri = 0; ri < 4; ++ri) rok[ri] = rowbase + 16 * (ri >> 1) + 8 * (ri & 1) < p.nrows;
  if (p.diag_on && p.diag_out && rowbase + p.row_off < cb + 64 && rowbase + p.row_off + 32 > cb) {  // diagonal tile (rare)
#pragma unroll
    for (int ri = 0; ri < 4; ++ri) {
      const int rg = rowbase + 16 * (ri >> 1) + 8 * (ri & 1);
      const int o = rg + p.row_off - cb;
      if (rok[ri] && o >= 0 && o < 64 && ((o >> 1) & 3) == t0) {
        float dv = 0.f;
#pragma unroll
        for (int rho = 0; rho < 8; ++rho)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            dv = (8 * rho + 2 * t0 + c == o) ? v[(ri >> 1) * 32 + rho * 4 + (ri & 1) * 2 + c] : dv;
        p.diag_out[rg] = dv * p.scale;
      }
    }
  }
  // self-masked launch (NT-Xent, reading N2): the warp's 32 rows meet their own column in this chunk
  const bool selfd = SELF && p.self_mask && rowbase + p.row_off < cb + 64 && rowbase + p.row_off + 32 > cb;
  const bool ragged = selfd || !(rok[0] && rok[1] && rok[2] && rok[3]) || cb + 64 > p.ncols;
  if (ragged) {  // masked entries -> -inf (k2 > 0 always: the host clamps it to FLT_MIN at s = 0, no -inf * 0)
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const int ri = (i >> 5) * 2 + ((i >> 1) & 1);
      const int col = cb + 8 * ((i >> 2) & 7) + 2 * t0 + (i & 1);
      const int row = rowbase + 16 * (ri >> 1) + 8 * (ri & 1);
      v[i] = (rok[ri] && col < p.ncols && !(selfd && col == row + p.row_off)) ? v[i] : -INFINITY;
    }
  }
  float ml[4];  // per-row local maxima (log2 units): 16 values per row through a tree of 3-input maxima
#pragma unroll
  for (int ri = 0; ri < 4; ++ri) {
    float x[16];
#pragma unroll
    for (int rho = 0; rho < 8; ++rho)
#pragma unroll
      for (int c = 0; c < 2; ++c) x[rho * 2 + c] = v[(ri >> 1) * 32 + rho * 4 + (ri & 1) * 2 + c];
#if INFCL_FWD_FMAX3
    const float a0 = fmax3(x[0], x[1], x[2]), a1 = fmax3(x[3], x[4], x[5]), a2 = fmax3(x[6], x[7], x[8]);
    const float a3 = fmax3(x[9], x[10], x[11]), a4 = fmax3(x[12], x[13], x[14]);
    const float mv = fmaxf(fmax3(a0, a1, a2), fmax3(a3, a4, x[15]));
#else  // A/B baseline: two-input maxima
    float mv = -INFINITY;
#pragma unroll
    for (int i = 0; i < 16; ++i) mv = fmaxf(mv, x[i]);
#endif
    ml[ri] = mv == -INFINITY ? -INFINITY : mv * k2;
  }
  // shared exponentials E = 2^{y - ml} (y = v * s * log2 e), row sums. Branch-free so the 4 rows'
  // exponentials interleave: an all-masked row uses reference 0 and its -inf logits give E = 0.
#pragma unroll
  for (int ri = 0; ri < 4; ++ri) {
    const float ref = ml[ri] == -INFINITY ? 0.f : ml[ri];
    const float2 kk = make_float2(k2, k2), nref = make_float2(-ref, -ref);
    float2 part[4];  // packed f32x2 arithmetic (FFMA2 / FADD2): half the ALU issue slots
#pragma unroll
    for (int rho = 0; rho < 8; ++rho) {
      float& x0 = v[(ri >> 1) * 32 + rho * 4 + (ri & 1) * 2];
      float& x1 = v[(ri >> 1) * 32 + rho * 4 + (ri & 1) * 2 + 1];
      const float2 t = __ffma2_rn(make_float2(x0, x1), kk, nref);
      if (rho < INFCL_FWD_POLY) {  // A/B variant: these exponentials on the FMA pipe (ex2_poly2)
        const float2 e = ex2_poly2(t);
        x0 = e.x;
        x1 = e.y;
      } else {
        x0 = ex2(t.x);
        x1 = ex2(t.y);
      }
      if (rho < 4) part[rho] = make_float2(x0, x1);
      else part[rho - 4] = __fadd2_rn(part[rho - 4], make_float2(x0, x1));
    }
    const float2 pa = __fadd2_rn(__fadd2_rn(part[0], part[1]), __fadd2_rn(part[2], part[3]));
    const float acc = pa.x + pa.y;
    const float mn = fmaxf(mrow[ri], ml[ri]);
    const float a_old = mrow[ri] == -INFINITY ? 0.f : ex2(mrow[ri] - mn);
    const float a_new = ml[ri] == -INFINITY ? 0.f : ex2(ml[ri] - mn);
    srow[ri] = (INFCL_MUTATION == 1 ? srow[ri] : srow[ri] * a_old) + acc * a_new;
    mrow[ri] = mn;
  }
  float Rw = fmaxf(fmaxf(ml[0], ml[1]), fmaxf(ml[2], ml[3]));
#pragma unroll
  for (int o = 16; o; o >>= 1) Rw = fmaxf(Rw, __shfl_xor_sync(0xffffffffu, Rw, o));
  float w[4];
#pragma unroll
  for (int ri = 0; ri < 4; ++ri) w[ri] = ml[ri] == -INFINITY ? 0.f : ex2(ml[ri] - Rw);
  float P[16];  // column partials over this thread's 4 rows: index rho*2 + c (the c pair packed)
#pragma unroll
  for (int rho = 0; rho < 8; ++rho) {
    float2 a = __fmul2_rn(make_float2(v[rho * 4], v[rho * 4 + 1]), make_float2(w[0], w[0]));
    a = __ffma2_rn(make_float2(v[rho * 4 + 2], v[rho * 4 + 3]), make_float2(w[1], w[1]), a);
    a = __ffma2_rn(make_float2(v[32 + rho * 4], v[32 + rho * 4 + 1]), make_float2(w[2], w[2]), a);
    a = __ffma2_rn(make_float2(v[32 + rho * 4 + 2], v[32 + rho * 4 + 3]), make_float2(w[3], w[3]), a);
    P[rho * 2] = a.x;
    P[rho * 2 + 1] = a.y;
  }
  // transposed butterfly over lane bits 4,3,2 -> lane holds columns 2*lane, 2*lane+1
#define XR16(O, N)                                                     \
  {                                                                    \
    const bool up = (lane & (O)) != 0;                                 \
    _Pragma("unroll") for (int i = 0; i < (N); ++i) {                  \
      const float send = up ? P[i] : P[i + (N)];                       \
      const float keep = up ? P[i + (N)] : P[i];                       \
      P[i] = keep + __shfl_xor_sync(0xffffffffu, send, (O));           \
    }                                                                  \
  }
  XR16(16, 8)
  XR16(8, 4)
  XR16(4, 2)
#undef XR16
  float S0 = P[0], S1 = P[1];
  float m0 = Rw, m1 = Rw;
  const bool bad = Rw != -INFINITY && ((cb + 2 * lane < p.ncols && S0 < 8.6736174e-19f) ||
                                       (cb + 2 * lane + 1 < p.ncols && S1 < 8.6736174e-19f));  // < 2^-60
  if (__any_sync(0xffffffffu, bad)) {
    // exact fallback (rare: a column far below the tile maximum): exact column max, second exponential
    float y[64];
    tmem_ld16x256x8(lchunk, y);
    tmem_ld16x256x8(lchunk + (16u << 16), y + 32);
    tmem_ld_wait();
    float cm[16];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const int ri = (i >> 5) * 2 + ((i >> 1) & 1);
      const int col = cb + 8 * ((i >> 2) & 7) + 2 * t0 + (i & 1);
      const int row = rowbase + 16 * (ri >> 1) + 8 * (ri & 1);
      y[i] = (rok[ri] && col < p.ncols && !(selfd && col == row + p.row_off)) ? y[i] * k2 : -INFINITY;
    }
#pragma unroll
    for (int rho = 0; rho < 8; ++rho)
#pragma unroll
      for (int c = 0; c < 2; ++c)
        cm[rho * 2 + c] = fmaxf(fmaxf(y[rho * 4 + c], y[rho * 4 + 2 + c]),
                                fmaxf(y[32 + rho * 4 + c], y[32 + rho * 4 + 2 + c]));
#define XM16(O, N)                                                     \
  {                                                                    \
    const bool up = (lane & (O)) != 0;                                 \
    _Pragma("unroll") for (int i = 0; i < (N); ++i) {                  \
      const float send = up ? cm[i] : cm[i + (N)];                     \
      const float keep = up ? cm[i + (N)] : cm[i];                     \
      cm[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, (O)));    \
    }                                                                  \
  }
    XM16(16, 8)
    XM16(8, 4)
    XM16(4, 2)
#undef XM16
    m0 = cm[0];
    m1 = cm[1];
#pragma unroll
    for (int rho = 0; rho < 8; ++rho) {
      const float c0 = __shfl_sync(0xffffffffu, m0, 4 * rho + t0);  // max of column 8rho+2t0
      const float c1 = __shfl_sync(0xffffffffu, m1, 4 * rho + t0);  // max of column 8rho+2t0+1
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float cc = c ? c1 : c0;
        float a = 0.f;
        if (cc != -INFINITY) {
          a = ex2(y[rho * 4 + c] - cc) + ex2(y[rho * 4 + 2 + c] - cc) + ex2(y[32 + rho * 4 + c] - cc) +
              ex2(y[32 + rho * 4 + 2 + c] - cc);
        }
        P[rho * 2 + c] = a;
      }
    }
#define XR16(O, N)                                                     \
  {                                                                    \
    const bool up = (lane & (O)) != 0;                                 \
    _Pragma("unroll") for (int i = 0; i < (N); ++i) {                  \
      const float send = up ? P[i] : P[i + (N)];                       \
      const float keep = up ? P[i + (N)] : P[i];                       \
      P[i] = keep + __shfl_xor_sync(0xffffffffu, send, (O));           \
    }                                                                  \
  }
    XR16(16, 8)
    XR16(8, 4)
    XR16(4, 2)
#undef XR16
    S0 = P[0];
    S1 = P[1];
  }
  return make_float4(m0, S0, m1, S1);
}

}  // namespace infcl
