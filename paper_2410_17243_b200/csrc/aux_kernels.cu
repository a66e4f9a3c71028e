// Small O(b)-work kernels around the fused pair kernel: LSE state merges (Eq.4 with the -inf identity,
// readings Q1/Q2, in the base-2 (m, sigma) form), LSE finalisation, the loss sum (Eq.2, fp64), the exact
// fp32 diagonal gradient term (reading H7) and the fp32 hi/lo bf16 split.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "kernels.h"

namespace infcl {

uint64_t& launch_counter() {
  static thread_local uint64_t n = 0;
  return n;
}

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ float2 merge_ms(float2 a, float2 b) {
  const float M = fmaxf(a.x, b.x);
  if (M == -INFINITY) return make_float2(-INFINITY, 0.f);
  return make_float2(M, a.y * exp2f(a.x - M) + b.y * exp2f(b.x - M));
}

// Mirror of the pair kernel's schedule (pair_kernel.cu, struct Sched): full waves W = n_rb / P, then the tail
// row blocks split into P contiguous ranges of T = R * n_ct items.
__device__ __forceinline__ long long tail_begin(long long T, int P, int p) { return (long long)p * T / P; }

__device__ int tail_pair_of(long long t, long long T, int P) {
  int p = (int)(((t + 1) * P + T - 1) / T) - 1;
  p = max(0, min(P - 1, p));
  while (p > 0 && tail_begin(T, P, p) > t) --p;
  while (p + 1 < P && tail_begin(T, P, p + 1) <= t) ++p;
  return p;
}

__global__ void init_state_kernel(float2* st, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) st[i] = make_float2(-INFINITY, 0.f);
}

__device__ __forceinline__ void merge_rows_body(int i, const float2* __restrict__ parts, float2* __restrict__ state,
                                                int nrows, int n_rb, int n_ct, int P, int rpp) {
  if (i >= nrows) return;
  const int rb = i / rpp;
  const int W = n_rb / P;
  float2 acc = state[i];
  if (rb < W * P) {
    acc = merge_ms(acc, parts[(long long)rb * rpp + (i % rpp)]);
  } else {
    const long long T = (long long)(n_rb - W * P) * n_ct;
    const long long t0 = (long long)(rb - W * P) * n_ct;
    const int p0 = tail_pair_of(t0, T, P), p1 = tail_pair_of(t0 + n_ct - 1, T, P);
    for (int p = p0; p <= p1; ++p)  // pairs with an empty tail range (T < P) wrote nothing
      if (tail_begin(T, P, p + 1) > tail_begin(T, P, p))
        acc = merge_ms(acc, parts[((long long)n_rb + p + (rb - W * P)) * rpp + (i % rpp)]);
  }
  state[i] = acc;
}

__global__ void merge_rows_kernel(const float2* __restrict__ parts, float2* __restrict__ state, int nrows, int n_rb,
                                  int n_ct, int P, int rpp) {
  merge_rows_body(blockIdx.x * blockDim.x + threadIdx.x, parts, state, nrows, n_rb, n_ct, P, rpp);
}

// Column state j merges the 2P per-CTA slot partials of column j (slots of pairs whose items never touched
// column j's tile hold stale data and are skipped).  Block = 32 columns x G slot groups: group g merges slots
// g, g+G, ... (independent loads in flight), then the G group partials merge in a fixed order (deterministic).
// G = 8 for wide passes (bandwidth-bound); G = 32 for the small blocks of a many-rank ring, where 8 groups left
// the GPU under-occupied and latency-bound (23 us for 8192 columns).  With no full wave (W = 0) the forward
// geometry has n_rb < P, so the tail bookkeeping fits 32-bit integers (64-bit kept for rectangular passes).
template <int COLS, int G>
__device__ __forceinline__ void merge_cols_body(int blk, const float2* __restrict__ slots, long long slot_ld,
                                                float2* __restrict__ state, int ncols, int n_rb, int n_ct, int P,
                                                int all_valid) {
  __shared__ float2 part[G][COLS];
  const int tx = threadIdx.x % COLS, g = threadIdx.x / COLS;
  const int j = blk * COLS + tx;
  const int W = n_rb / P;
  const bool check = !(all_valid || W > 0);
  const long long T = check ? (long long)n_rb * n_ct : 0;
  const bool small = T * P < (1LL << 31);  // always for the square forward passes: n_ct <= n_rb < P
  float2 acc = make_float2(-INFINITY, 0.f);
  if (j < ncols && !check) {  // every slot holds data: unconditional loads, four in flight per thread
    int sl = g;
    for (; sl + 3 * G < 2 * P; sl += 4 * G) {
      const float2 v0 = __ldg(slots + (long long)sl * slot_ld + j);
      const float2 v1 = __ldg(slots + (long long)(sl + G) * slot_ld + j);
      const float2 v2 = __ldg(slots + (long long)(sl + 2 * G) * slot_ld + j);
      const float2 v3 = __ldg(slots + (long long)(sl + 3 * G) * slot_ld + j);
      acc = merge_ms(merge_ms(merge_ms(merge_ms(acc, v0), v1), v2), v3);  // same order as one at a time
    }
    for (; sl < 2 * P; sl += G) acc = merge_ms(acc, __ldg(slots + (long long)sl * slot_ld + j));
  } else if (j < ncols) {
    const int ct = j / kColsPerTile;
    for (int sl = g; sl < 2 * P; sl += G) {
      const int p = sl >> 1;
      bool visited;
      if (small) {
        const int a = p * (int)T / P, e = (p + 1) * (int)T / P;
        visited = (e - a >= n_ct) || (e > a && a + ((ct - a % n_ct) % n_ct + n_ct) % n_ct < e);
      } else {
        const long long a = tail_begin(T, P, p), e = tail_begin(T, P, p + 1);
        visited = (e - a >= n_ct) || (e > a && a + ((ct - a % n_ct) % n_ct + n_ct) % n_ct < e);
      }
      if (visited) acc = merge_ms(acc, __ldg(slots + (long long)sl * slot_ld + j));
    }
  }
  part[g][tx] = acc;
  __syncthreads();
  if (g == 0 && j < ncols) {
    float2 a = state[j];
#pragma unroll
    for (int k = 0; k < G; ++k) a = merge_ms(a, part[k][tx]);
    state[j] = a;
  }
}

template <int COLS, int G>
__global__ void __launch_bounds__(256) merge_cols_kernel(const float2* __restrict__ slots, long long slot_ld,
                                                         float2* __restrict__ state, int ncols, int n_rb, int n_ct,
                                                         int P, int all_valid) {
  merge_cols_body<COLS, G>(blockIdx.x, slots, slot_ld, state, ncols, n_rb, n_ct, P, all_valid);
}

// One ring step's two merges in one launch: blocks [0, nbr) fold the step's row partials into the row state
// (merge_rows), the rest fold the per-CTA column slots into the travelling column state (merge_cols).
template <int COLS, int G>
__global__ void __launch_bounds__(256) merge_step_kernel(const float2* __restrict__ parts, float2* __restrict__ rstate,
                                                         int nrows, int rn_rb, int rn_ct, int rP, int rpp, int nbr,
                                                         const float2* __restrict__ slots, long long slot_ld,
                                                         float2* __restrict__ cstate, int ncols, int n_rb, int n_ct,
                                                         int P) {
  if ((int)blockIdx.x < nbr) {
    merge_rows_body(blockIdx.x * 256 + threadIdx.x, parts, rstate, nrows, rn_rb, rn_ct, rP, rpp);
  } else {
    merge_cols_body<COLS, G>(blockIdx.x - nbr, slots, slot_ld, cstate, ncols, n_rb, n_ct, P, 0);
  }
}

// End of the forward: r_i, c_i from the row / column states, and the rank's loss partial
// sum_i (r_i + c_i - 2 x_ii) (fp64, block reduction + one atomic per block): finalize x2 + loss_partial fused.
__global__ void __launch_bounds__(256) fwd_finish_kernel(const float2* __restrict__ rst, const float2* __restrict__ cst,
                                                         float* __restrict__ r, float* __restrict__ c,
                                                         const float* __restrict__ diag, int n, double* acc) {
  double v = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float2 a = rst[i], b = cst[i];
    const float ri = (a.x == -INFINITY ? -INFINITY : a.x + log2f(a.y)) * 0.69314718055994531f;
    const float ci = (b.x == -INFINITY ? -INFINITY : b.x + log2f(b.y)) * 0.69314718055994531f;
    r[i] = ri;
    c[i] = ci;
    v += (double)ri + (double)ci - 2.0 * (double)diag[i];
  }
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __shared__ double ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < 8 ? ws[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) atomicAdd(acc, v);
  }
}

// Backward tail: the row blocks the last wave splits between CTA pairs are drained by each pair into its own
// scratch slot (plain stores); this kernel adds the slots of each row to dst in ascending pair order, so the
// gradients are bitwise reproducible (a red.add per pair would add them in completion order).  Slot of
// (pair p, tail row block rb) = p + rb - W*P (as the forward's row partials); one block per row.
__global__ void tail_combine_kernel(const float4* __restrict__ scratch, float* __restrict__ dst, int ld_dst,
                                    int nrows, int d_out, int n_rb, int n_ct, int P, int rpp) {
  // one block per tail row: the row block's sharing pairs are found once (thread 0), the threads stream the row
  __shared__ int sp[2];
  const int W = n_rb / P;
  const long long row = (long long)W * P * rpp + blockIdx.x;
  if (row >= nrows) return;
  const int rb = (int)(row / rpp);
  const long long T = (long long)(n_rb - W * P) * n_ct;
  if (threadIdx.x == 0) {
    const long long t0 = (long long)(rb - W * P) * n_ct;
    sp[0] = tail_pair_of(t0, T, P);
    sp[1] = tail_pair_of(t0 + n_ct - 1, T, P);
  }
  __syncthreads();
  const int p0 = sp[0], p1 = sp[1], d4 = d_out >> 2;
  float4* o = reinterpret_cast<float4*>(dst + row * ld_dst);
  for (int k4 = threadIdx.x; k4 < d4; k4 += blockDim.x) {
    float4 a = o[k4];
    for (int p = p0; p <= p1; ++p) {
      if (tail_begin(T, P, p + 1) <= tail_begin(T, P, p)) continue;  // empty range: no slot written
      const float4 v = __ldg(scratch + ((long long)(p + rb - W * P) * rpp + (row % rpp)) * d4 + k4);
      a.x += v.x;
      a.y += v.y;
      a.z += v.z;
      a.w += v.w;
    }
    o[k4] = a;
  }
}

__global__ void loss_write_kernel(const double* acc, float* loss, double inv2b) { *loss = (float)(*acc * inv2b); }

__global__ void set_scalar_kernel(float* dst, float v) { *dst = v; }

__global__ void sum_f64_kernel(const double* in, int n, double* out) {
  double v = 0.0;
  for (int i = 0; i < n; ++i) v += in[i];
  *out = v;
}

__global__ void scale_log2_kernel(const float* __restrict__ x, float* __restrict__ y, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] * 1.4426950408889634f;
}

// dA_i += s * g/(2b) * (e^{x_ii - r_i} + e^{x_ii - c_i} - 2) * B_i   (exact fp32 diagonal term, H7)
// exact fp32 diagonal term of Eq.7 (reading H7): dA_i (+)= coef * g * (P_ii + Q_ii - 2) * B_i.  One warp per row,
// 16-byte stores (d % 8 == 0 and ld % 8 == 0 keep every row 32-B aligned).  init = 1 writes the term (the
// backward's accumulator initialisation, replacing a memset and a later read-modify-write); init = 0 adds it.
__global__ void diag_term_kernel(float* __restrict__ dA, int ld_dA, const void* __restrict__ B, int ldB, int b_f32,
                                 const float* __restrict__ diag, const float* __restrict__ r,
                                 const float* __restrict__ c, const float* __restrict__ grad, float coef_base, int n,
                                 int d, int init) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const int lane = threadIdx.x & 31;
  const float x = diag[i];
  float w = coef_base * grad[0] * (expf(x - r[i]) + expf(x - c[i]) - 2.f);
  if (INFCL_MUTATION == 4) w = 0.f;
  float4* out = reinterpret_cast<float4*>(dA + (long long)i * ld_dA);
  for (int k4 = lane; k4 < (d >> 2); k4 += 32) {
    float4 bv;
    if (b_f32) {
      bv = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(B) + (long long)i * ldB)[k4];
    } else {
      const uint2 raw = reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(B) + (long long)i * ldB)[k4];
      const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
      const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
      bv = make_float4(lo.x, lo.y, hi.x, hi.y);
    }
    float4 o = init ? make_float4(0.f, 0.f, 0.f, 0.f) : out[k4];
    o.x += w * bv.x;
    o.y += w * bv.y;
    o.z += w * bv.z;
    o.w += w * bv.w;
    out[k4] = o;
  }
}

// fp32 -> [hi | hi | lo] (mode 0) or [hi | lo | hi] (mode 1) bf16 rows of width 3d: I'.T'^T = hi.hi + hi.lo + lo.hi
__global__ void split_f32_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, int n, int d,
                                 int mode) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n * d) return;
  const long long i = idx / d;
  const int k = (int)(idx % d);
  const float v = x[idx];
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
  __nv_bfloat16* o = out + i * 3 * d;
  o[k] = hi;
  o[d + k] = mode == 0 ? hi : lo;
  o[2 * d + k] = mode == 0 ? lo : hi;
}

// out = in[:, 0:d] + in[:, d:2d] (mode 0) or in[:, 0:d] + in[:, 2d:3d] (mode 1)
__global__ void combine_f32_kernel(const float* __restrict__ in, int ld_in, float* __restrict__ out, int n, int d,
                                   int mode) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n * d) return;
  const long long i = idx / d;
  const int k = (int)(idx % d);
  const float* row = in + i * ld_in;
  out[idx] = row[k] + row[(mode == 0 ? d : 2 * d) + k];
}

// sum_i <dI_i, I_i> * inv_s in fp64 (the logit-scale gradient identity)
__global__ void grad_scale_kernel(const void* __restrict__ I, int i_f32, const float* __restrict__ dI, long long n,
                                  double inv_s, double* out) {
  double v = 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const float x = i_f32 ? reinterpret_cast<const float*>(I)[k]
                          : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(I)[k]);
    v += (double)x * (double)dI[k];
  }
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __shared__ double ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) atomicAdd(out, v * inv_s);
  }
}

void launch_grad_scale(const void* I, int i_f32, const float* dI, long long n, double inv_s, double* out,
                       cudaStream_t s) {
  grad_scale_kernel<<<std::min(nblk(n, 256), 1184u), 256, 0, s>>>(I, i_f32, dI, n, inv_s, out);
  ++launch_counter();
}

void launch_init_state(float2* st, int n, cudaStream_t s) {
  init_state_kernel<<<nblk(n, 256), 256, 0, s>>>(st, n);
  ++launch_counter();
}
void launch_merge_rows(const float2* parts, float2* state, int nrows, const PassGeom& g, cudaStream_t s) {
  merge_rows_kernel<<<nblk(nrows, 256), 256, 0, s>>>(parts, state, nrows, g.n_rb, g.n_ct, g.npairs, g.rpp);
  ++launch_counter();
}
void launch_merge_cols(const float2* slots, long long slot_ld, float2* state, int ncols, const PassGeom& g,
                       cudaStream_t s, bool all_valid) {
  // 32 columns x 8 slot groups for wide merges (bandwidth-bound); 8 columns x 32 groups below 32768 columns,
  // where 8 groups left the GPU under-occupied and latency-bound (23 us for 8192 columns)
  if (ncols >= 32768)
    merge_cols_kernel<32, 8><<<nblk(ncols, 32), 256, 0, s>>>(slots, slot_ld, state, ncols, g.n_rb, g.n_ct, g.npairs,
                                                             all_valid ? 1 : 0);
  else
    merge_cols_kernel<8, 32><<<nblk(ncols, 8), 256, 0, s>>>(slots, slot_ld, state, ncols, g.n_rb, g.n_ct, g.npairs,
                                                            all_valid ? 1 : 0);
  ++launch_counter();
}
void launch_merge_step(const float2* parts, float2* rstate, int nrows, const float2* slots, long long slot_ld,
                       float2* cstate, int ncols, const PassGeom& g, cudaStream_t s) {
  const unsigned nbr = nblk(nrows, 256);
  if (ncols >= 32768)
    merge_step_kernel<32, 8><<<nbr + nblk(ncols, 32), 256, 0, s>>>(parts, rstate, nrows, g.n_rb, g.n_ct, g.npairs,
                                                                   g.rpp, (int)nbr, slots, slot_ld, cstate, ncols,
                                                                   g.n_rb, g.n_ct, g.npairs);
  else
    merge_step_kernel<8, 32><<<nbr + nblk(ncols, 8), 256, 0, s>>>(parts, rstate, nrows, g.n_rb, g.n_ct, g.npairs,
                                                                  g.rpp, (int)nbr, slots, slot_ld, cstate, ncols,
                                                                  g.n_rb, g.n_ct, g.npairs);
  ++launch_counter();
}
void launch_fwd_finish(const float2* rstate, const float2* cstate, float* r, float* c, const float* diag, int n,
                       double* acc, cudaStream_t s) {
  fwd_finish_kernel<<<std::min(nblk(n, 256), 592u), 256, 0, s>>>(rstate, cstate, r, c, diag, n, acc);
  ++launch_counter();
}
void launch_tail_combine(const float* scratch, float* dst, int ld_dst, int nrows, int d_out, const PassGeom& g,
                         cudaStream_t s) {
  const int W = g.n_rb / g.npairs;
  const long long rows = (long long)nrows - (long long)W * g.npairs * g.rpp;
  if (rows <= 0) return;
  const int threads = std::min(256, std::max(32, (d_out / 4 + 31) / 32 * 32));
  tail_combine_kernel<<<(unsigned)rows, threads, 0, s>>>(reinterpret_cast<const float4*>(scratch), dst, ld_dst,
                                                         nrows, d_out, g.n_rb, g.n_ct, g.npairs, g.rpp);
  ++launch_counter();
}
void launch_loss_write(const double* acc, float* loss, int64_t b, cudaStream_t s) {
  loss_write_kernel<<<1, 1, 0, s>>>(acc, loss, 0.5 / (double)b);
  ++launch_counter();
}
void launch_set_scalar(float* dst, float v, cudaStream_t s) {
  set_scalar_kernel<<<1, 1, 0, s>>>(dst, v);
  ++launch_counter();
}
void launch_sum_f64(const double* in, int n, double* out, cudaStream_t s) {
  sum_f64_kernel<<<1, 1, 0, s>>>(in, n, out);
  ++launch_counter();
}
void launch_scale_log2(const float* x, float* y, int n, cudaStream_t s) {
  scale_log2_kernel<<<nblk(n, 256), 256, 0, s>>>(x, y, n);
  ++launch_counter();
}
void launch_diag_term(float* dA, int ld_dA, const void* B, int ldB, int dtype_f32, const float* diag, const float* r,
                      const float* c, const float* grad, float coef_base, int n, int d, bool init, cudaStream_t s) {
  if (n <= 0) return;
  diag_term_kernel<<<nblk(n, 8), 256, 0, s>>>(dA, ld_dA, B, ldB, dtype_f32, diag, r, c, grad, coef_base, n, d,
                                              init ? 1 : 0);
  ++launch_counter();
}
void launch_split_f32(const float* x, void* out, int n, int d, int mode, cudaStream_t s) {
  split_f32_kernel<<<nblk((long long)n * d, 256), 256, 0, s>>>(x, reinterpret_cast<__nv_bfloat16*>(out), n, d, mode);
  ++launch_counter();
}
void launch_combine_f32(const float* in, int ld_in, float* out, int n, int d, int mode, cudaStream_t s) {
  combine_f32_kernel<<<nblk((long long)n * d, 256), 256, 0, s>>>(in, ld_in, out, n, d, mode);
  ++launch_counter();
}

}  // namespace infcl
