// Hardware self-test of the UMMA building blocks the loss kernels use: TMA (SW128) -> smem -> tcgen05.mma
// (1 CTA or CTA pair, K-major or MN-major A) -> TMEM, dumped raw so tests can verify the data layout.
#include <cuda.h>
#include <cuda_runtime.h>

#include "../host_utils.h"
#include "../../../include/infcl_diag.h"
#include "../ptx.cuh"

namespace infcl {

template <int NCTA>
__global__ void __launch_bounds__(128, 1)
    probe_umma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                      int N, int K, int a_mn, int fmt, float* out, int ncols) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int Mc = M / NCTA, Nc = N / NCTA, KB = K / 64;
  uint8_t* sA = smem;
  uint8_t* sB = smem + KB * Mc * 128;
  __shared__ uint64_t bar_full, bar_done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t cta = NCTA == 2 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar_full, 1);
    mbar_init(&bar_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<NCTA>(&tmem_base, 512);
  tc_fence_before();
  if constexpr (NCTA == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;

  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)(KB * (Mc + Nc) * 128);
    if (cta == 0) mbar_arrive_expect_tx(&bar_full, bytes * NCTA);
    for (int kb = 0; kb < KB; ++kb) {
      if (!a_mn) {
        void* dst = sA + kb * Mc * 128;
        if constexpr (NCTA == 2) tma_load_2d_pair(dst, &tmA, &bar_full, kb * 64, cta * Mc);
        else tma_load_2d(dst, &tmA, &bar_full, kb * 64, 0);
      } else {
        for (int mb = 0; mb < Mc / 64; ++mb) {
          void* dst = sA + (kb * (Mc / 64) + mb) * 8192;
          if constexpr (NCTA == 2) tma_load_2d_pair(dst, &tmA, &bar_full, cta * Mc + mb * 64, kb * 64);
          else tma_load_2d(dst, &tmA, &bar_full, mb * 64, kb * 64);
        }
      }
      void* dstb = sB + kb * Nc * 128;
      if constexpr (NCTA == 2) tma_load_2d_pair(dstb, &tmB, &bar_full, kb * 64, cta * Nc);
      else tma_load_2d(dstb, &tmB, &bar_full, kb * 64, 0);
    }
  }
  if (cta == 0 && threadIdx.x == 32) {
    mbar_wait(&bar_full, 0);
    tc_fence_after();
    // fmt bit 0 / bit 1: A / B holds fp16 (format 0 in the instruction descriptor) instead of bf16 (format 1)
    const uint32_t idesc = idesc_bf16(M, N, a_mn, 0) & ~((fmt & 1) ? (7u << 7) : 0u) & ~((fmt & 2) ? (7u << 10) : 0u);
    for (int k = 0; k < K / 16; ++k) {
      uint64_t ad = a_mn ? smem_desc_sw128(smem_u32(sA + (k / 4) * (Mc / 64) * 8192 + (k % 4) * 2048), 8192, 1024)
                         : smem_desc_sw128(smem_u32(sA + (k / 4) * Mc * 128 + (k % 4) * 32), 16, 1024);
      uint64_t bd = smem_desc_sw128(smem_u32(sB + (k / 4) * Nc * 128 + (k % 4) * 32), 16, 1024);
      umma_bf16<NCTA>(tbase, ad, bd, idesc, k > 0);
    }
    if constexpr (NCTA == 2) umma_commit_pair_mc(&bar_done, 0x3);
    else umma_commit_1cta(&bar_done);
  }
  mbar_wait(&bar_done, 0);
  tc_fence_after();
  float v[32];
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < ncols; c0 += 32) {
    tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 32 && c0 + j < ncols; ++j) out[((size_t)cta * 128 + row) * ncols + c0 + j] = v[j];
  }
  tc_fence_before();
  if constexpr (NCTA == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) tmem_dealloc<NCTA>(tbase, 512);
}

}  // namespace infcl

using namespace infcl;

extern "C" infcl_status infcl_probe_umma(const void* A, const void* B, int M, int N, int K, int a_mn_major, int ncta,
                                         int fmt, float* out, int ncols, void* stream) {
  if (!A || !B || !out) return fail(INFCL_ERR_INVALID_ARG, "null pointer");
  if (ncta != 1 && ncta != 2) return fail(INFCL_ERR_INVALID_ARG, "ncta must be 1 or 2");
  if (K % 64 || K > 256 || M % (64 * ncta) || N % (16 * ncta) || ncols % 32 || ncols > 512)
    return fail(INFCL_ERR_SHAPE, "probe shape");
  const int Mc = M / ncta, Nc = N / ncta;
  CUtensorMap ta, tb;
  infcl_status st = a_mn_major ? make_tmap_bf16(&ta, A, K, M, M, 64, 64) : make_tmap_bf16(&ta, A, M, K, K, 64, Mc);
  if (st) return st;
  if ((st = make_tmap_bf16(&tb, B, N, K, K, 64, Nc))) return st;
  size_t smem = 1024 + (size_t)(K / 64) * (Mc + Nc) * 128;
  cudaStream_t s = (cudaStream_t)stream;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncta);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ncta;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (ncta == 1) {
    INFCL_CUDA_TRY(cudaFuncSetAttribute(probe_umma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    INFCL_CUDA_TRY(cudaLaunchKernelEx(&cfg, probe_umma_kernel<1>, ta, tb, M, N, K, a_mn_major, fmt, out, ncols));
  } else {
    INFCL_CUDA_TRY(cudaFuncSetAttribute(probe_umma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    INFCL_CUDA_TRY(cudaLaunchKernelEx(&cfg, probe_umma_kernel<2>, ta, tb, M, N, K, a_mn_major, fmt, out, ncols));
  }
  return INFCL_OK;
}

// ------------------------------------------------------------------ TS layout self-test (A in TMEM)
// CTA pair, D (128 x 256) = A (128 x K) * B (K x 256): CTA c's 4 warps write A rows [64c, 64c+64) into TMEM
// columns 256.. in the duplicated 2x2 layout (warp q: lanes 32q.., rows 32 (q & 1) + lane; bf16 pairs packed low
// element first), B is TMA-loaded per CTA as its 128 N columns (two 64-wide MN-major SW128 boxes of K rows), the
// leader issues K/16 TS MMAs into TMEM column 0, and the raw TMEM image (128 lanes x 128 columns) is dumped.
namespace infcl {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe_umma_ts_kernel(const __grid_constant__ CUtensorMap tmB, const uint16_t* A, int K, int mode, float* out) {
  const bool b_km = (mode & 1) != 0;  // B K-major ([256][K] rows, 64-wide K boxes) instead of MN-major ([K][256])
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_full, bar_done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t cta = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bar_full, 1);
    mbar_init(&bar_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<2>(&tmem_base, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t box = (uint32_t)K * 128;  // one 64-column MN-major box of K rows
  if (threadIdx.x == 0) {
    if (cta == 0) mbar_arrive_expect_tx(&bar_full, 2 * 2 * box);
    if (b_km) {  // K blocks of 64: box 64 K x 128 rows (this CTA's N half) = 16 KB each
      for (int kb = 0; kb < K / 64; ++kb) tma_load_2d_pair(smem + kb * 16384, &tmB, &bar_full, kb * 64, (int)cta * 128);
    } else {
      for (int h = 0; h < 2; ++h) tma_load_2d_pair(smem + h * box, &tmB, &bar_full, (int)cta * 128 + h * 64, 0);
    }
  }
  {
    const int row = (int)cta * 64 + 32 * (warp & 1) + lane;
    for (int c0 = 0; c0 < K / 2; c0 += 32) {
      uint32_t r[32];
      for (int i = 0; i < 32; ++i) r[i] = (uint32_t)A[(size_t)row * K + 2 * (c0 + i)] |
                                          ((uint32_t)A[(size_t)row * K + 2 * (c0 + i) + 1] << 16);
      tmem_st32(tbase + ((uint32_t)(warp * 32) << 16) + 256 + c0, r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (cta == 0 && warp == 1) {
    mbar_wait(&bar_full, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_bf16(128, 256, 0, b_km ? 0 : 1);
    for (int k = 0; k < K / 16; ++k) {
      const uint64_t bd = b_km ? smem_desc_sw128(smem_u32(smem) + (k / 4) * 16384 + (k % 4) * 32, 16, 1024)
                               : smem_desc_sw128(smem_u32(smem) + k * 2048, box, 1024);
      umma_ts_pair_warp(tbase, tbase + 256 + 8 * k, bd, idesc, k > 0);
    }
    umma_commit_pair_mc_warp(&bar_done, 0x3);
  }
  mbar_wait(&bar_done, 0);
  tc_fence_after();
  float v[32];
  const int l = warp * 32 + lane;
  for (int c0 = 0; c0 < 128; c0 += 32) {
    tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[((size_t)cta * 128 + l) * 128 + c0 + j] = v[j];
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) tmem_dealloc<2>(tbase, 512);
}
}  // namespace infcl

extern "C" infcl_status infcl_probe_umma_ts(const void* A, const void* B, int K, int mode, float* out, void* stream) {
  if (!A || !B || !out) return fail(INFCL_ERR_INVALID_ARG, "null pointer");
  if (K % 64 || K > 256) return fail(INFCL_ERR_SHAPE, "probe shape");
  CUtensorMap tb;
  // B [K][256] row-major: box 64 features x K rows; or (mode & 1) B [256][K]: box 64 K x 128 rows
  infcl_status st = (mode & 1) ? make_tmap_bf16(&tb, B, 256, K, K, 64, 128) : make_tmap_bf16(&tb, B, K, 256, 256, 64, K);
  if (st) return st;
  const size_t smem = 1024 + (size_t)4 * K * 128;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  INFCL_CUDA_TRY(cudaFuncSetAttribute(probe_umma_ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  INFCL_CUDA_TRY(cudaLaunchKernelEx(&cfg, probe_umma_ts_kernel, tb, reinterpret_cast<const uint16_t*>(A), K, mode, out));
  return INFCL_OK;
}

// ------------------------------------------------------------------ MMA issue-rate microbenchmark
// Operands resident in smem (contents irrelevant), one thread of the leader CTA issues `iters` back-to-back
// MMAs of the given shape, then commits; cycles per MMA are measured on the issuing SM.
namespace infcl {
__device__ __forceinline__ bool lane_is_zero() { return (threadIdx.x & 31) == 0; }
template <int NCTA>
__global__ void __launch_bounds__(128, 1) probe_rate_kernel(int M, int N, int a_mn, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_done, bar_ready, bar_dummy, bar_done2;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  const uint32_t cta = NCTA == 2 ? cluster_ctarank() : 0;
  const bool stream = (a_mn & 128) != 0;  // M=128 N=256 pair loop over the pair kernel's real footprint (192 KB)
  const uint32_t fillv = (iters & (1 << 30)) ? 0x3c003c00u : 0x3f803f80u;  // iters bit 30: the walk probes' fill
  // iters bit 29: the idle warps wait in the cluster barrier (as the walk probes' idle warps do) instead of on an
  // mbarrier while the MMA warp issues
  const bool idle_cluster_bar = (iters & (1 << 29)) != 0;
  iters &= (1 << 29) - 1;
  for (int i = threadIdx.x; i < (stream ? 192 : 64) * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = fillv;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar_done, 1);
    mbar_init(&bar_ready, 1);
    mbar_init(&bar_dummy, 1 << 19);
    mbar_init(&bar_done2, 1);
    fence_mbar_init();
    mbar_arrive(&bar_ready);  // phase 0 completes: waits on it return at once
  }
  if (warp == 1) tmem_alloc<NCTA>(&tmem_base, 512);
  tc_fence_before();
  if constexpr (NCTA == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  __shared__ volatile int stop_flag;
  if (threadIdx.x == 0) stop_flag = 0;
  __syncthreads();
  const int ld_mode = (a_mn >> 5) & 3;  // 1: warps 2-3 stream tcgen05.ld 16x256b; 2: 32x32b; from TMEM cols 256+
  if (ld_mode && (warp == 2 || warp == 3)) {
    float sink = 0.f;
    float v[32];
    while (!stop_flag) {
#pragma unroll 1
      for (int rep = 0; rep < 16; ++rep) {
        const uint32_t ta = tbase + ((uint32_t)(warp * 32) << 16) + 256 + (rep & 3) * 32;
        if (ld_mode == 1) tmem_ld16x256x8(ta, v);
        else tmem_ld32(ta, v);
        tmem_ld_wait();
        sink += v[rep & 31];
      }
    }
    if (sink == 12345.f) out[2] = 1;
  }
  if (cta == 0 && warp == 1) {  // whole warp converged, elect.sync inside the asm (as in pair_kernel)
    const uint32_t idesc = idesc_bf16(M, N, a_mn & 1, 0);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    const int G = (a_mn & 31) >= 2 ? ((a_mn & 31) >> 1) : 0;  // every G MMAs: barrier wait + fence, commit
    const int amn = a_mn & 1;
    const uint64_t ad0 = amn ? smem_desc_sw128(sa, 8192, 1024) : smem_desc_sw128(sa, 16, 1024);
    const uint64_t bd0 = smem_desc_sw128(sb, 16, 1024);
    const uint64_t astep = amn ? 128 : 2;
    const long long t0 = clock64();
    if (stream) {  // A: 8 boxes of 64 rows x 128 B (64 KB), B: 4 stages of 2 boxes of 128 rows x 128 B (128 KB)
      const uint32_t sA = smem_u32(smem), sB = smem_u32(smem + 65536);
      // G field in this mode = loop-structure variant bits: 1 first MMA of every 4 stages overwrites (accumulate 0),
      // 2 D rotates over 4 buffers of 128 columns every 4 stages, 4 tcgen05.fence::after_thread_sync every stage
      // (an earlier build: D alternating between two regions every stage -- 64 cycles), 8 commit to a real
      // (count-1) barrier every stage and a wait 3 stages back
      const int var = G;
      uint32_t ph = 0;
      for (int i = 0; i < iters; i += 8) {
        const int s8 = i >> 3, st = s8 & 3;
        const uint32_t acc = ((var & 1) && st == 0) ? 0u : 1u;
        uint32_t d = tbase;
        if (var & 2) d += (uint32_t)((s8 >> 2) & 3) * 128;
        if (var & 4) tc_fence_after();  // (variant bit 4 now: tcgen05.fence::after_thread_sync per stage)
        umma_stage_pair<true, (8192 >> 4), (16384 >> 4)>(d, (uint32_t)smem_desc_sw128(sA + 2 * st * 8192, 16, 1024),
                                                         (uint32_t)smem_desc_sw128(sB + st * 32768, 16, 1024), idesc, acc);
        if (var & 8) {
          umma_commit_pair_mc_warp(&bar_done2, 0x3);
          if (s8 >= 3) {  // wait for the commit 3 stages back (a 4-deep ring's empty barrier)
            mbar_wait(&bar_done2, ph);
            ph ^= 1;
          }
        }
      }
    } else if (G == 0) {
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) umma_bf16_warp<NCTA>(tbase, ad0 + (uint64_t)((k & 3) * astep), bd0 + (uint64_t)(2 * (k & 3)), idesc, 1u);
      }
    } else {
      for (int i = 0; i < iters; i += 8) {
        mbar_wait(&bar_ready, 0);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k) umma_bf16_warp<NCTA>(tbase, ad0 + (uint64_t)((k & 3) * astep), bd0 + (uint64_t)(2 * (k & 3)), idesc, 1u);
        if constexpr (NCTA == 2) umma_commit_pair_mc_warp(&bar_dummy, 0x3);
      }
    }
    const long long t1 = clock64();
    if constexpr (NCTA == 2) umma_commit_pair_mc_warp(&bar_done, 0x3);
    else if (lane_is_zero()) umma_commit_1cta(&bar_done);
    mbar_wait(&bar_done, 0);
    const long long t2 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
    stop_flag = 1;
  }
  if (NCTA == 2 && cta != 0 && threadIdx.x == 0) stop_flag = 1;
  if ((cta != 0 || warp != 1) && !idle_cluster_bar) mbar_wait(&bar_done, 0);
  tc_fence_before();
  if constexpr (NCTA == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) tmem_dealloc<NCTA>(tbase, 512);
}
}  // namespace infcl

extern "C" infcl_status infcl_probe_mma_rate(int M, int N, int a_mn_major, int ncta, int iters, long long* out_cycles,
                                             void* stream) {
  if (!out_cycles || (ncta != 1 && ncta != 2) || iters < 1) return fail(INFCL_ERR_INVALID_ARG, "bad probe args");
  cudaLaunchConfig_t cfg = {};
  const int nclusters = (a_mn_major >> 8) > 0 ? (a_mn_major >> 8) : 1;  // bits 8+: clusters launched concurrently
  a_mn_major &= 0xff;
  cfg.gridDim = dim3(ncta * nclusters);
  cfg.blockDim = dim3(128);
  const bool stream_mode = (a_mn_major & 128) != 0;
  cfg.dynamicSmemBytes = (stream_mode ? 192 : 64) * 1024 + 1024;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ncta;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (ncta == 1) {
    INFCL_CUDA_TRY(cudaFuncSetAttribute(probe_rate_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65 * 1024));
    INFCL_CUDA_TRY(cudaLaunchKernelEx(&cfg, probe_rate_kernel<1>, M, N, a_mn_major, iters, out_cycles));
  } else {
    INFCL_CUDA_TRY(cudaFuncSetAttribute(probe_rate_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 193 * 1024));
    INFCL_CUDA_TRY(cudaLaunchKernelEx(&cfg, probe_rate_kernel<2>, M, N, a_mn_major, iters, out_cycles));
  }
  return INFCL_OK;
}

// co-resident cluster count for a 1-CTA-per-SM kernel (diagnostic; not part of the ABI)
extern "C" int infcl_diag_max_clusters(int cluster) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster * 64);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(probe_rate_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (cluster > 8) cudaFuncSetAttribute(probe_rate_kernel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int n = -1;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_rate_kernel<1>, &cfg);
  return e == cudaSuccess ? n : -(int)e;
}

// ------------------------------------------------------------------ TMA streaming-throughput microbenchmark
// Every CTA streams `iters` 16-KB (or 32-KB) stages through a ring of 6 smem stages; a consumer thread releases
// each stage as soon as it lands.  mode 0: two 2D boxes [64 x 64 rows]; 1: one 2D box [64 x 128 rows];
// 2: one 3D box (64, 64 rows, 2 column blocks); 3: one 2D box [64 x 256 rows] (32-KB stage).
namespace infcl {
__global__ void __launch_bounds__(64, 1)
    probe_tma_kernel(const __grid_constant__ CUtensorMap t2a, const __grid_constant__ CUtensorMap t2b,
                     const __grid_constant__ CUtensorMap t3, int mode, int iters, int nrows, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int NS = 6;
  __shared__ uint64_t full[NS], empty[NS];
  const int stage_bytes = mode == 3 ? 32768 : 16384;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    int s = 0;
    uint32_t ph = 0;
    int row = (blockIdx.x * 997) % (nrows - 256);
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      uint8_t* dst = smem + s * 32768;
      const int col = (i & 7) * 64;
      if (mode == 0) {
        tma_load_2d(dst, &t2a, &full[s], col, row);
        tma_load_2d(dst + 8192, &t2a, &full[s], col, row + 64);
      } else if (mode == 1) {
        tma_load_2d(dst, &t2b, &full[s], col, row);
      } else if (mode == 2) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
            "[%2];" ::"r"(smem_u32(dst)),
            "l"(reinterpret_cast<uint64_t>(&t3)), "r"(smem_u32(&full[s])), "r"(0), "r"(row), "r"((i & 3) * 2)
            : "memory");
      } else {
        tma_load_2d(dst, &t2b, &full[s], col, row);
        tma_load_2d(dst + 16384, &t2b, &full[s], col, row + 128);
      }
      row += 256;
      if (row >= nrows - 256) row -= nrows - 512;
      if (++s == NS) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[s], ph);
      mbar_arrive(&empty[s]);
      if (++s == NS) {
        s = 0;
        ph ^= 1;
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}
}  // namespace infcl

extern "C" int infcl_diag_tma_rate(const void* X, int nrows, int d, int mode, int iters, int nblocks, long long* out) {
  CUtensorMap a, b, c;
  if (make_tmap_bf16(&a, X, nrows, d, d, 64, 64) || make_tmap_bf16(&b, X, nrows, d, d, 64, 128)) return -1;
  // 3D view: (64 inner elements, rows, column blocks of 64) with strides (row: d*2 B, block: 128 B)
  {
    typedef CUresult (*Fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    cuuint64_t dims[3] = {64, (cuuint64_t)nrows, (cuuint64_t)(d / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)d * 2, 128};
    cuuint32_t box[3] = {64, 64, 2};
    cuuint32_t es[3] = {1, 1, 1};
    if (reinterpret_cast<Fn>(p)(&c, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(X), dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -2;
  }
  cudaFuncSetAttribute(probe_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 1024);
  probe_tma_kernel<<<nblocks, 64, 6 * 32768 + 1024>>>(a, b, c, mode, iters, nrows, out);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -3;
}

// ------------------------------------------------------------------ S-GEMM loop-structure probe (diagnostic)
// One CTA pair issues `tiles` S tiles of the forward shape (M=128 pair, N=256, K = 64*KB) through the same
// umma_stage_pair path as pair_kernel, with optional features switched on by `mode` bits, to find which part
// of the real loop costs tensor throughput:  1: walk A over KB boxes (else reuse box 0);  2: walk B over
// `ns` 32-KB stages (else reuse stage 0);  4: rotate 4 TMEM accumulators per tile (else one);  8: commit each
// stage to a per-stage barrier and wait it `ns` stages later (ring back-pressure without TMA).
namespace infcl {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe_walk_kernel(int tiles, int KB, int ns, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sA = smem_raw;
  uint8_t* sB = smem_raw + KB * 8192;
  __shared__ __align__(8) uint64_t ring[16], done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  const uint32_t cta = cluster_ctarank();
  for (int i = threadIdx.x; i < (KB * 8192 + ns * 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem_raw)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&ring[i], 1);
    mbar_init(&done, ((mode & 524288) && !(mode & 32)) ? 2 : 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<2>(&tmem_base, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (cta == 0 && warp == 1) {
    const uint32_t idS = idesc_bf16(128, 256, 0, 0);
    const int KC = KB / 2;
    int stage = 0;
    uint32_t ph = 0;
    long long n_stage_total = 0;
    const long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dS = tbase + ((mode & 4) ? (t & 3) * 128 : 0);
      for (int kc = 0; kc < KC; ++kc) {
        if ((mode & 8) && n_stage_total >= ns) {  // the slot's previous use must have completed
          mbar_wait(&ring[stage], ph ^ 1);
        }
        tc_fence_after();
        const uint32_t a = smem_u32(sA + ((mode & 1) ? 2 * kc * 8192 : 0));
        const uint32_t b = smem_u32(sB + ((mode & 2) ? stage * 32768 : 0));
        const uint64_t ad0 = smem_desc_sw128(a, 16, 1024), bd0 = smem_desc_sw128(b, 16, 1024);
        umma_stage_pair<true, (8192 >> 4), (16384 >> 4)>(dS, (uint32_t)ad0, (uint32_t)bd0, idS, kc != 0);
        if (mode & 8) umma_commit_pair_mc_warp(&ring[stage], 0x1);
        ++n_stage_total;
        if (++stage == ns) {
          stage = 0;
          ph ^= 1;
        }
      }
    }
    const long long t1 = clock64();
    umma_commit_pair_mc_warp(&done, 0x3);
    mbar_wait(&done, 0);
    const long long t2 = clock64();
    if (threadIdx.x == 32) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  if (cta != 0 && warp == 1) mbar_wait(&done, 0);
  tc_fence_before();
  cluster_sync();
  if (warp == 1) tmem_dealloc<2>(tbase, 512);
}
}  // namespace infcl

extern "C" int infcl_diag_walk(int tiles, int KB, int ns, int mode, long long* out) {
  const size_t smem = (size_t)KB * 8192 + (size_t)ns * 32768;
  if (cudaFuncSetAttribute(infcl::probe_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))
    return -1;
  infcl::probe_walk_kernel<<<2, 128, smem>>>(tiles, KB, ns, mode, out);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -3;
}

// Second loop-structure probe with the real kernel's warp roles (320 threads): warp 9 issues (leader CTA),
// warp 8 = producer (waits empty[s], arrives full[s]; no TMA), warps 0-7 = epilogue stand-ins (wait sfull[b],
// tcgen05.ld one 32x32b chunk if mode & 64, arrive sfree[b] on the leader).  mode bits: 16 producer ring,
// 32 epilogue handshake (4 TMEM buffers).  Grid = 2 * nclusters CTAs.
namespace infcl {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    probe_walk2_kernel(int tiles, int KB, int ns, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sA = smem_raw;
  const bool wide = (mode & 512) != 0;  // M=256 pair MMAs (128 rows per CTA), 2 TMEM buffers of 256 columns
  uint8_t* sB = smem_raw + KB * (wide ? 16384 : 8192);
  __shared__ __align__(8) uint64_t full[16], empty[16], sfull[4], sfree[4], done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  for (int i = threadIdx.x; i < (KB * (wide ? 16384 : 8192) + ns * 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem_raw)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sfree[i], 16);
    }
    mbar_init(&done, ((mode & 524288) && !(mode & 32)) ? 2 : 1);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<2>(&tmem_base, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const int KC = KB / 2;
  const long long nst = (long long)tiles * KC;
  // mode 524288: TWO issuing warps (9 and 7, different SM sub-partitions) take alternate ring stages (each waits for
  // and commits its own stages; results invalid -- both accumulate into the same D -- timing only)
  const bool two = (mode & 524288) != 0 && !(mode & 32);
  if ((warp == 9 || (two && warp == 7)) && cta == 0) {
    const int me = warp == 7 ? 1 : 0;
    const bool st = (mode & 2048) != 0;  // S^T shape: M=256 (stage rows) x N=128 (sA rows), same bytes per stage
    const uint32_t idS = st ? idesc_bf16(256, 128, 0, 0) : idesc_bf16(wide ? 256 : 128, 256, 0, 0);
    int stage = 0;
    uint32_t ph = 0, sfph = 0;
    long long n = 0;
    const long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const int buf = wide ? (t & 1) : (t & 3);
      if (mode & 32) {
        mbar_wait_cluster(&sfree[buf], ((sfph >> buf) & 1u) ^ 1u);
        sfph ^= 1u << buf;
      }
      if (!(mode & 8192)) tc_fence_after();
      // bisection bits: 8192 no tcgen05 fences, 16384 fixed D, 32768 always accumulate, 65536 no per-stage commits
      const uint32_t dS = (mode & 16384) ? tbase : tbase + buf * (wide ? 256 : 128);
      for (int kc = 0; kc < KC; ++kc) {
        if (two && (int)(n & 1) != me) {  // the other issuer's stage
          ++n;
          if (++stage == ns) {
            stage = 0;
            ph ^= 1;
          }
          continue;
        }
        if (mode & 16) mbar_wait(&full[stage], ph);
        else if (n >= ns && !(mode & 128)) mbar_wait(&empty[(mode & 1024) ? (stage & ~1) : stage], ph ^ 1);
        if (!(mode & 8192)) tc_fence_after();
        const uint32_t acc = (mode & 32768) ? 1u : (kc != 0 ? 1u : 0u);
        const uint64_t ad0 = smem_desc_sw128(smem_u32(sA + 2 * kc * (wide ? 16384 : 8192)), 16, 1024);
        const uint64_t bd0 = smem_desc_sw128(smem_u32(sB + stage * 32768), 16, 1024);
        if (wide) umma_stage_pair<true, (16384 >> 4), (16384 >> 4)>(dS, (uint32_t)ad0, (uint32_t)bd0, idS, acc);
        else if (st) umma_stage_pair<true, (16384 >> 4), (8192 >> 4)>(dS, (uint32_t)bd0, (uint32_t)ad0, idS, acc);
        else if (mode & 4096)  // TS form: A (garbage) in TMEM columns 384.., B = the stage as an MN-major operand
          umma_stage_dI_ts_pair(dS, tbase + 384, (uint32_t)smem_desc_sw128(smem_u32(sB + stage * 32768), 16384, 1024),
                                idesc_bf16(128, 256, 0, 1), acc);
        else if (mode & 131072) {  // issue style L: 8 single-MMA asm statements, 64-bit descriptors from C++
#pragma unroll
          for (int k = 0; k < 8; ++k)
            umma_bf16_warp<2>(dS, ad0 + (uint64_t)((k >> 2) * (8192 >> 4) + 2 * (k & 3)),
                              bd0 + (uint64_t)((k >> 2) * (16384 >> 4) + 2 * (k & 3)), idS, k == 0 ? acc : 1u);
        } else if (mode & 262144) {  // issue style E: one elected lane issues all 8 (plain asm), then the warp syncs
          uint32_t el;
          asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(el));
          if (el) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              umma_bf16<2>(dS, ad0 + (uint64_t)((k >> 2) * (8192 >> 4) + 2 * (k & 3)),
                           bd0 + (uint64_t)((k >> 2) * (16384 >> 4) + 2 * (k & 3)), idS, k == 0 ? acc : 1u);
          }
          __syncwarp();
        } else umma_stage_pair<true, (8192 >> 4), (16384 >> 4)>(dS, (uint32_t)ad0, (uint32_t)bd0, idS, acc);
        if (mode & 65536) {
          // no per-stage commits (only with mode 128: nothing waits for them)
        } else if (mode & 1024) {  // ONE commit per two stages: empty[even] covers the pair
          if (stage & 1) umma_commit_pair_mc_warp(&empty[stage - 1], 0x3);
        } else if (!(mode & 256)) {
          umma_commit_pair_mc_warp(&empty[stage], 0x3);
        } else if (stage & 1) {  // release two stages per commit pair, issued back to back at the odd stage
          umma_commit_pair_mc_warp(&empty[stage - 1], 0x3);
          umma_commit_pair_mc_warp(&empty[stage], 0x3);
        }
        ++n;
        if (++stage == ns) {
          stage = 0;
          ph ^= 1;
        }
      }
      if (mode & 32) umma_commit_pair_mc_warp(&sfull[buf], 0x3);
    }
    const long long t1 = clock64();
    umma_commit_pair_mc_warp(&done, 0x3);
    mbar_wait(&done, 0);
    const long long t2 = clock64();
    if (lane == 0 && blockIdx.x == 0 && warp == 9) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  } else if (warp == 8 && (mode & 16)) {
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (long long n = 0; n < nst; ++n) {
        if (!(mode & 1024) || !(stage & 1)) mbar_wait(&empty[(mode & 1024) ? (stage & ~1) : stage], ph ^ 1);
        if (cta == 0) mbar_arrive(&full[stage]);
        if (++stage == ns) {
          stage = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp < 8 && (mode & 32)) {
    uint32_t sph = 0;
    float sink = 0.f;
    for (int t = 0; t < tiles; ++t) {
      const int buf = wide ? (t & 1) : (t & 3);
      mbar_wait(&sfull[buf], (sph >> buf) & 1u);
      sph ^= 1u << buf;
      tc_fence_after();
      if (mode & 64) {
        float v[32];
        tmem_ld32(tbase + ((uint32_t)((warp & 3) * 32) << 16) + buf * (wide ? 256 : 128) + (warp >> 2) * 32, v);
        tmem_ld_wait();
        sink += v[lane];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&sfree[buf], 0);
    }
    if (sink == 1234.5f) out[3] = 1;
  }
  if (!(warp == 9 && cta == 0) && warp == 9) mbar_wait(&done, 0);
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 9) tmem_dealloc<2>(tbase, 512);
}
}  // namespace infcl

extern "C" int infcl_diag_walk2(int tiles, int KB, int ns, int mode, int nclusters, long long* out) {
  const size_t smem = (size_t)KB * ((mode & 512) ? 16384 : 8192) + (size_t)ns * 32768;
  if (cudaFuncSetAttribute(infcl::probe_walk2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))
    return -1;
  infcl::probe_walk2_kernel<<<2 * nclusters, 320, smem>>>(tiles, KB, ns, mode, out);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -3;
}

// ------------------------------------------------------------------ TMA path probe 2 (diagnostic)
// Per-SM streaming rate of a ring of `ns` 32-KB stages (consumer releases on arrival), by copy flavour:
// mode 0: two 2D tensor boxes [64 x 128 rows] SW128 (the kernels' path); mode 1: two 1D bulk copies of 16 KB
// (cp.async.bulk, contiguous source = pre-swizzled tile images); mode 2: one 1D bulk copy of 32 KB.
namespace infcl {
__global__ void __launch_bounds__(64, 1)
    probe_tma2_kernel(const __grid_constant__ CUtensorMap tb, const uint8_t* src, long long src_bytes, int nrows,
                      int mode, int ns, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full[8], empty[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    int s = 0;
    uint32_t ph = 0;
    int row = (blockIdx.x * 997) % (nrows - 256);
    long long off = ((long long)blockIdx.x * 1000003LL * 16) % (src_bytes - 65536);
    off &= ~15LL;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], 32768);
      uint8_t* dst = smem_raw + s * 32768;
      if (mode == 0) {
        const int col = (i & 7) * 64;
        tma_load_2d(dst, &tb, &full[s], col, row);
        tma_load_2d(dst + 16384, &tb, &full[s], col, row + 128);
        row += 256;
        if (row >= nrows - 256) row -= nrows - 512;
      } else {
        const int pieces = mode == 1 ? 2 : 1, sz = 32768 / pieces;
        for (int k = 0; k < pieces; ++k)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(dst + k * sz)),
              "l"(src + off + k * sz), "r"(sz), "r"(smem_u32(&full[s]))
              : "memory");
        off += 32768;
        if (off + 32768 > src_bytes) off = 0;
      }
      if (++s == ns) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[s], ph);
      mbar_arrive(&empty[s]);
      if (++s == ns) {
        s = 0;
        ph ^= 1;
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}
}  // namespace infcl

extern "C" int infcl_diag_tma_rate2(const void* X, int nrows, int d, int mode, int ns, int iters, int nblocks,
                                    long long* out) {
  CUtensorMap b;
  if (make_tmap_bf16(&b, X, nrows, d, d, 64, 128)) return -1;
  if (ns < 1 || ns > 6) return -2;
  cudaFuncSetAttribute(infcl::probe_tma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  infcl::probe_tma2_kernel<<<nblocks, 64, 6 * 32768>>>(b, static_cast<const uint8_t*>(X), (long long)nrows * d * 2,
                                                         nrows, mode, ns, iters, out);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -3;
}

// ------------------------------------------------------------------ TMA path probe 3 (diagnostic)
// Is the ~75 B/clk per-SM streaming cap an SM-ingress limit or an L2-egress limit?  Clusters of 2 CTAs stream
// 32-KB stages (two 2D SW128 boxes of [64 x 128 rows]).  mode 0: each CTA loads both boxes itself; mode 1: CTA r
// loads box r with .multicast::cluster to both CTAs (each SM still receives 32 KB per stage, L2 sends half).
// The peer's consumer must free a stage before it is refilled, so `empty` takes one arrival from each CTA.
namespace infcl {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1)
    probe_tma3_kernel(const __grid_constant__ CUtensorMap tb, int nrows, int mode, int ns, int iters,
                      long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const uint32_t cta = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], mode == 1 ? 2 : 1);
    }
    fence_mbar_init();
  }
  cluster_sync();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    int s = 0;
    uint32_t ph = 0;
    int row = ((blockIdx.x >> (mode == 1 ? 1 : 0)) * 997) % (nrows - 256);
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], 32768);
      uint8_t* dst = smem_raw + s * 32768;
      const int col = (i & 7) * 64;
      if (mode == 0) {
        tma_load_2d(dst, &tb, &full[s], col, row);
        tma_load_2d(dst + 16384, &tb, &full[s], col, row + 128);
      } else {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], "
            "[%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst + cta * 16384)),
            "l"(reinterpret_cast<uint64_t>(&tb)), "r"(smem_u32(&full[s])), "r"(col), "r"(row + (int)cta * 128),
            "h"((uint16_t)0x3)
            : "memory");
      }
      row += 256;
      if (row >= nrows - 256) row -= nrows - 512;
      if (++s == ns) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[s], ph);
      mbar_arrive(&empty[s]);
      if (mode == 1) mbar_arrive_cluster(&empty[s], cta ^ 1u);
      if (++s == ns) {
        s = 0;
        ph ^= 1;
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  cluster_sync();
}
}  // namespace infcl

extern "C" int infcl_diag_tma_rate3(const void* X, int nrows, int d, int mode, int ns, int iters, int nblocks,
                                    long long* out) {
  CUtensorMap b;
  if (make_tmap_bf16(&b, X, nrows, d, d, 64, 128)) return -1;
  if (ns < 1 || ns > 6 || (nblocks & 1)) return -2;
  cudaFuncSetAttribute(infcl::probe_tma3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  infcl::probe_tma3_kernel<<<nblocks, 64, 6 * 32768>>>(b, nrows, mode, ns, iters, out);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -3;
}

// ------------------------------------------------------------------ copy-path probe (diagnostic)
// The IPC ring transport's copy (cudaMemcpyAsync device to device); only mode 0 exists.
extern "C" int infcl_diag_copy(void* dst, const void* src, size_t bytes, int mode, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (mode != 0) return (int)cudaErrorInvalidValue;
  return (int)cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st);
}

// ------------------------------------------------------------------ L2 reduction throughput (single-pass feasibility)
// The single-pass backward of Alg.4 would flush a per-tile fp32 dT partial (256 columns x d) into a
// global dT that all CTA pairs of a column-synchronous wave share.  This probe measures how fast 148 SMs can
// reduce fp32 data into global memory.  Each CTA holds `chunk_bytes` of fp32 ones in smem and adds them `iters`
// times into `dst` (dst_floats floats, the "column tile" window):
//   mode 0: cp.reduce.async.bulk .add.f32 (one thread, 16-KB bulk ops), every CTA at the same window offset
//           (worst-case address contention: all pairs reduce the same tile at once);
//   mode 1: the same, CTA b at offset (it + b) * chunk (same window, staggered);
//   mode 2: the same, disjoint windows per CTA (dst_floats must hold nblocks windows of chunk_bytes);
//   mode 3: red.global.add.v4.f32 from every thread (staggered like mode 1).
// Bytes reduced = nblocks * iters * chunk_bytes; the caller times the launch.
namespace infcl {
__global__ void __launch_bounds__(256, 1) probe_reduce_kernel(float* dst, long long dst_floats, int chunk_bytes,
                                                              int iters, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* src = reinterpret_cast<float*>(smem_raw);
  const int nf = chunk_bytes / 4;
  for (int i = threadIdx.x; i < nf; i += blockDim.x) src[i] = 1.0f;
  fence_proxy_async_smem();
  __syncthreads();
  const long long win = mode == 2 ? dst_floats / gridDim.x : dst_floats;
  float* base = mode == 2 ? dst + (long long)blockIdx.x * win : dst;
  const long long slots = win / nf;
  if (mode <= 2) {
    if (threadIdx.x == 0) {
      for (int it = 0; it < iters; ++it) {
        const long long slot = mode == 1 ? (it + blockIdx.x) % slots : it % slots;
        float* d = base + slot * nf;
        for (int off = 0; off < chunk_bytes; off += 16384) {
          const int sz = min(16384, chunk_bytes - off);
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                           reinterpret_cast<char*>(d) + off),
                       "r"(smem_u32(smem_raw + off)), "r"(sz)
                       : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else {
    for (int it = 0; it < iters; ++it) {
      const long long slot = (it + blockIdx.x) % slots;
      float* d = base + slot * nf;
      for (int i = threadIdx.x * 4; i < nf; i += blockDim.x * 4) {
        const float4 v = *reinterpret_cast<const float4*>(src + i);
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d + i), "f"(v.x), "f"(v.y), "f"(v.z),
                     "f"(v.w)
                     : "memory");
      }
    }
  }
}
}  // namespace infcl

extern "C" int infcl_diag_reduce_rate(float* dst, long long dst_floats, int chunk_bytes, int iters, int nblocks, int mode,
                                      void* stream) {
  if (!dst || chunk_bytes < 16 || chunk_bytes % 16 || chunk_bytes > 196608 || iters < 1 || nblocks < 1 || mode < 0 ||
      mode > 3)
    return -1;
  const long long win = mode == 2 ? dst_floats / nblocks : dst_floats;
  if (win < chunk_bytes / 4) return -2;
  if (cudaFuncSetAttribute(infcl::probe_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk_bytes) !=
      cudaSuccess)
    return -3;
  infcl::probe_reduce_kernel<<<nblocks, 256, chunk_bytes, (cudaStream_t)stream>>>(dst, dst_floats, chunk_bytes, iters,
                                                                                    mode);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

extern "C" const char* infcl_diag_last_error(void) { return infcl::last_error_string(); }
