// Internal (C++) interface between the ABI layer (api.cu) and the CUDA kernels.
#pragma once
// INFCL_MUTATION (test builds only, scripts/mutation_check.py): 1 = forward row merge drops the rescale of the
// old running sum; 2 = backward G loses its column term; 3 = wide forward streams the wrong B column tile;
// 4 = the exact diagonal gradient term is skipped.  The parity suite must fail for each; 0 = the product.
#ifndef INFCL_MUTATION
#define INFCL_MUTATION 0
#endif
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/infcl.h"

namespace infcl {

constexpr int kRowsPerPair = 128;  // stationary rows per CTA pair (64 per SM)
constexpr int kColsPerTile = 256;  // streamed columns per tile (128 per SM)
constexpr int kMaxD = 768;         // TMEM budget: 128 (S) + 3 x 128 (dA^T chunks) columns

// One "pass" of the pair kernel over (stationary A rows) x (streamed B block).
struct PassArgs {
  const void* A;        // [nrows][ld] bf16 stationary side (I for fwd / dI pass, T for the dT pass)
  const void* B;        // [ncols][ld] bf16 streamed block
  int nrows, ncols;     // valid rows of A and B
  int dk, ld;           // K extent (feature dim) and row stride in elements
  float scale;          // s
  int diag_on;          // B is A's own block: the positive pair of row i is column i + row_off
  int row_off;          // diagonal: the positive pair of local row i is local column i + row_off
  int slots_merge;      // forward: column slots are pre-initialised (-inf, 0); always merge into them
  int self_mask;        // column i + row_off is row i's own view: excluded from LSEs and G (NT-Xent, N2)
  // forward outputs (per pass / ring step)
  float2* col_slots;    // [2 * npairs][slot_ld] (m2, sigma) partials (workspace)
  long long slot_ld;
  float2* row_parts;    // [(n_rb + npairs) * 128] row partials (workspace)
  float* diag_out;      // [nrows] x_ii (natural units) or nullptr
  // backward
  const float* lse_row2;  // [nrows] row LSE in log2 units (r * log2 e)
  const float* lse_col2;  // [ncols] column LSE in log2 units
  float* dA;              // [nrows][ld_dA] fp32, accumulated with red.add
  int ld_dA, d_out;
  const float* grad;      // device scalar g
  float coef_base;        // s / (2 b)
  float* tail_scratch;    // [2 npairs - 1][128][d_out] fp32: per-pair partials of split tail row blocks (workspace),
                          // added in pair order by launch_tail_combine (deterministic); nullptr = red.add
  // fused backward (launch_pair_backward_fused): the column side's gradient and the G ring workspace
  float* dB;              // [ncols][ld_dB] fp32, accumulated with red.add (dB = coef * G^T A)
  int ld_dB;
  void* gc_ws;            // gc_plan(nrows, ncols, dk).bytes: step counters, then the G ring
  size_t gc_ws_bytes;
};

// fused backward plan (pair_kernel.cu gc_plan): ok = the fused kernel applies (bf16 K width <= 512, >= 2 pairs)
struct GcPlan {
  bool ok;
  int npairs, pp, pc, ring;
  long long n_steps, n_ctr;
  size_t ctr_bytes, bytes;
};
GcPlan gc_plan(int nrows, int ncols, int dk);
// three-role fused backward (fused3.cu): producers (S, G), dI readers, dT readers; d <= 512
struct Gc3Plan {
  bool ok;
  int npairs, pp, pc, ring, n_rb, n_ct;
  long long n_steps, n_ctr;
  size_t ctr_bytes, bytes;
};
Gc3Plan gc3_plan(int nrows, int ncols, int dk);
infcl_status launch_bwd3(const PassArgs& a, cudaStream_t s);

struct PassGeom {
  int n_rb, n_ct, npairs;
  long long n_items;
  int rpp;  // stationary rows per CTA pair: 128 (narrow pair kernel) or 256 (wide forward kernel)
};

PassGeom pass_geom(int nrows, int ncols);  // narrow pair kernel (backward; forward with INFCL_FWD_NARROW)
PassGeom wide_geom(int nrows, int ncols);  // wide forward kernel
PassGeom fwd_geom(int nrows, int ncols);   // geometry of the forward kernel launch_pair_forward uses
bool wide_forward_enabled();
infcl_status launch_pair_forward(const PassArgs& a, cudaStream_t s);  // wide forward unless INFCL_FWD_NARROW
infcl_status launch_wide_forward(const PassArgs& a, cudaStream_t s);
infcl_status launch_pair_backward(const PassArgs& a, cudaStream_t s);
// single-pass backward: dA and dB from one launch (producer pairs: S, G, dA; consumer pairs: dB from the G ring)
infcl_status launch_pair_backward_fused(const PassArgs& a, cudaStream_t s);
// launch bookkeeping shared by the pair kernels (pair_kernel.cu)
cudaEvent_t profile_begin(cudaStream_t s);
void profile_end(int kind, cudaEvent_t e0, cudaStream_t s);
unsigned long long* debug_buffer(cudaStream_t s);  // INFCL_DEBUG_WAITS accumulators (zeroed) or nullptr
unsigned long long* debug_buffer_ptr();             // the same buffer (10 x 16 counters), not re-zeroed
// prod_pairs (fused backward): CTA pairs [0, prod_pairs) are producers, the rest consumers
void debug_report(const char* name, int npairs, cudaStream_t s, int prod_pairs = -1);

// auxiliary kernels (aux_kernels.cu)
void launch_init_state(float2* st, int n, cudaStream_t s);
void launch_merge_rows(const float2* row_parts, float2* row_state, int nrows, const PassGeom& g, cudaStream_t s);
void launch_merge_cols(const float2* col_slots, long long slot_ld, float2* col_state, int ncols, const PassGeom& g,
                       cudaStream_t s, bool all_valid = false);
// one ring step's row merge (rows [0, nrows) of rstate) and column merge (cstate) in one launch; g = the
// step's forward geometry (square pass: the same geometry indexes both)
void launch_merge_step(const float2* parts, float2* rstate, int nrows, const float2* slots, long long slot_ld,
                       float2* cstate, int ncols, const PassGeom& g, cudaStream_t s);
// r, c from the row / column states and the rank's loss partial into acc (finalize x2 + loss partial fused)
void launch_fwd_finish(const float2* rstate, const float2* cstate, float* r, float* c, const float* diag, int n,
                       double* acc, cudaStream_t s);
void launch_loss_write(const double* acc, float* loss, int64_t b, cudaStream_t s);
// dst rows of the backward's split tail row blocks += their per-pair scratch partials, in ascending pair order
void launch_tail_combine(const float* scratch, float* dst, int ld_dst, int nrows, int d_out, const PassGeom& g,
                         cudaStream_t s);
void launch_scale_log2(const float* x, float* y, int n, cudaStream_t s);
void launch_set_scalar(float* dst, float v, cudaStream_t s);
void launch_sum_f64(const double* in, int n, double* out, cudaStream_t s);  // out = in[0] + ... + in[n-1], in order
// exact diagonal gradient term; init = true writes it (accumulator initialisation), false adds it
void launch_diag_term(float* dA, int ld_dA, const void* B, int ldB, int dtype_f32, const float* diag, const float* r,
                      const float* c, const float* grad, float coef_base, int n, int d, bool init, cudaStream_t s);
void launch_split_f32(const float* x, void* out_bf16, int n, int d, int mode, cudaStream_t s);
void launch_grad_scale(const void* I, int i_f32, const float* dI, long long n, double inv_s, double* out,
                       cudaStream_t s);
void launch_combine_f32(const float* in, int ld_in, float* out, int n, int d, int mode, cudaStream_t s);

uint64_t& launch_counter();
void profile_enable(bool on);
infcl_status profile_read(int kind, int* launches, double* total_ms);

}  // namespace infcl
