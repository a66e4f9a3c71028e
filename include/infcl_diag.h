/*
 * infcl_diag.h -- hardware probes and microbenchmarks of the B200 building blocks the Inf-CL kernels use.
 *
 * NOT part of the product ABI (include/infcl.h): these live in a separate library, libinfcl_diag.so, that
 * only tests/test_gpu_probe.py and scripts/experiments/ load.  The product library libinfcl.so exports exactly
 * the symbols infcl.h declares (checked by tests/test_abi.py); this header lists exactly what
 * libinfcl_diag.so exports.  Every pointer is DEVICE memory unless stated; calls are not thread-safe.
 * Status-returning probes report details through infcl_diag_last_error().  Integer-returning probes return 0
 * on success and a negative code on a bad argument or launch failure.
 */
#ifndef INFCL_DIAG_H_
#define INFCL_DIAG_H_

#include <stddef.h>
#include <stdint.h>

#include "infcl.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Detail of the last failing status-returning probe on this thread. */
const char* infcl_diag_last_error(void);

/* UMMA layout self-test: D = A * B^T for one tile, A [M][K] (a_mn_major = 0) or stored as [K][M] (a_mn_major = 1),
 * B [N][K]; ncta = 1 or 2 (CTA pair); fmt bit 0 / bit 1: A / B elements are fp16 (else bf16), i.e. the
 * instruction descriptor's a_format / b_format fields of tcgen05.mma.kind::f16.  Writes the raw TMEM image
 * out[ncta][128 lanes][ncols] (fp32).  K % 64 == 0, K <= 256, ncols % 32 == 0, ncols <= 512. */
infcl_status infcl_probe_umma(const void* A, const void* B, int M, int N, int K, int a_mn_major, int ncta, int fmt,
                              float* out, int ncols, void* stream);

/* TS layout self-test (A operand in TMEM): D (128 x 256) = A (128 x K) * B (K x 256) on a CTA pair, A bf16 [128][K]
 * row-major (written into TMEM by the CTAs in the duplicated 2x2 layout), B bf16 [K][256] row-major (MN-major
 * operand; mode & 1: B bf16 [256][K], K-major).  Writes the raw TMEM image out[2][128 lanes][128 columns] (fp32).  K % 64 == 0, K <= 256. */
infcl_status infcl_probe_umma_ts(const void* A, const void* B, int K, int mode, float* out, void* stream);

/* MMA issue-rate probe: one CTA (pair) issues `iters` back-to-back tcgen05.mma (bf16, K=16) of shape M x N from
 * resident smem; out_cycles (device, 2 x int64) = {issue cycles, issue-to-completion cycles}.  a_mn_major bits:
 * 0 = MN-major A, 1-4 = barrier wait + commit every G MMAs, 5-6 = concurrent TMEM-load warps, 8+ = clusters. */
infcl_status infcl_probe_mma_rate(int M, int N, int a_mn_major, int ncta, int iters, long long* out_cycles,
                                  void* stream);

/* Co-resident cluster count of a 1-CTA-per-SM kernel with 200 KB of smem for cluster size `cluster`
 * (negative cudaError_t on failure). */
int infcl_diag_max_clusters(int cluster);

/* TMA streaming-throughput probes over X [nrows][d] bf16: `nblocks` CTAs stream `iters` stages each (modes and
 * ring depth `ns` as documented in csrc/diag/probe.cu); out = per-CTA cycle counts (device int64). */
int infcl_diag_tma_rate(const void* X, int nrows, int d, int mode, int iters, int nblocks, long long* out);
int infcl_diag_tma_rate2(const void* X, int nrows, int d, int mode, int ns, int iters, int nblocks, long long* out);
int infcl_diag_tma_rate3(const void* X, int nrows, int d, int mode, int ns, int iters, int nblocks, long long* out);

/* Loop-structure probes of the pair kernel's ring handshakes (tiles x KB K-blocks through an ns-stage ring,
 * 74 CTA pairs or `nclusters`); out = cycle counts (device int64). */
int infcl_diag_walk(int tiles, int KB, int ns, int mode, long long* out);
int infcl_diag_walk2(int tiles, int KB, int ns, int mode, int nclusters, long long* out);

/* Copy-path probe (scripts/experiments/overlap_probe.py): device-to-device copy of `bytes` on `stream`;
 * mode 0 = cudaMemcpyAsync (the IPC ring transport's copy); any other mode returns cudaErrorInvalidValue.
 * Returns the cudaError_t of the enqueue (0 = success). */
int infcl_diag_copy(void* dst, const void* src, size_t bytes, int mode, void* stream);

/* L2 reduction-throughput probe (single-pass backward feasibility): `nblocks` CTAs each add
 * `chunk_bytes` of fp32 ones from smem into dst (dst_floats floats) `iters` times.  mode 0: cp.reduce.async.bulk
 * .add.f32, all CTAs at the same offset; 1: the same, staggered offsets; 2: disjoint per-CTA windows;
 * 3: red.global.add.v4.f32 from every thread, staggered.  Asynchronous on `stream`; the caller times it. */
int infcl_diag_reduce_rate(float* dst, long long dst_floats, int chunk_bytes, int iters, int nblocks, int mode,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* INFCL_DIAG_H_ */
