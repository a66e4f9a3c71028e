// Hardware self-test of the UMMA building blocks the loss kernels use: TMA (SW128) -> smem -> tcgen05.mma
// (1 CTA or CTA pair, K-major or MN-major A) -> TMEM, dumped raw so tests can verify the data layout.
#include <cuda.h>
#include <cuda_runtime.h>

#include "host_utils.h"
#include "ptx.cuh"

namespace infcl {

template <int NCTA>
__global__ void __launch_bounds__(128, 1)
    probe_umma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                      int N, int K, int a_mn, float* out, int ncols) {
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
    const uint32_t idesc = idesc_bf16(M, N, a_mn, 0);
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
                                         float* out, int ncols, void* stream) {
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
    INFCL_CUDA_TRY(cudaLaunchKernelEx(&cfg, probe_umma_kernel<1>, ta, tb, M, N, K, a_mn_major, out, ncols));
  } else {
    INFCL_CUDA_TRY(cudaFuncSetAttribute(probe_umma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    INFCL_CUDA_TRY(cudaLaunchKernelEx(&cfg, probe_umma_kernel<2>, ta, tb, M, N, K, a_mn_major, out, ncols));
  }
  return INFCL_OK;
}
