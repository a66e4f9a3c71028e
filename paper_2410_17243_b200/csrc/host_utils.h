// Host-side helpers shared by the library translation units: error state, TMA tensor maps.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/infcl.h"

namespace infcl {

void set_last_error(const std::string& msg);
infcl_status fail(infcl_status st, const std::string& msg);
const char* last_error_string();  // this thread's detail (infcl_last_error / infcl_diag_last_error)

#define INFCL_CUDA_TRY(expr)                                                                   \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess)                                                                     \
      return ::infcl::fail(INFCL_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// 2D bf16 tensor map over a row-major [rows][cols] matrix with row stride `ld` elements, box
// [box_cols (inner) x box_rows], 128-byte swizzle, zero fill out of bounds.
// fp32 row-major [rows][ld] (ld in elements), box box_rows x box_cols, 128-B swizzle (box_cols * 4 == 128)
infcl_status make_tmap_f32_sw128(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                                 uint32_t box_cols, uint32_t box_rows);
infcl_status make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                            uint32_t box_cols, uint32_t box_rows);

int num_sms();
// CTA pairs the persistent pair kernels may occupy: num_sms() / 2, minus this thread's carve-out (SMs left free for
// the NCCL ring transport's kernels, PairCarveOut), capped by INFCL_PAIRS (diagnostic)
int max_pairs();
struct PairCarveOut {  // RAII: leave `pairs` CTA pairs free while a ring call enqueues its kernels (this thread)
  explicit PairCarveOut(int pairs);
  ~PairCarveOut();
  int saved;
};

}  // namespace infcl
