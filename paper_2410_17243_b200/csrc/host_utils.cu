// Host helpers: thread-local error detail, status strings, TMA tensor-map encoding via the driver entry
// point (no link-time dependency on libcuda, so the library loads on a GPU-less host).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "host_utils.h"

namespace infcl {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

infcl_status fail(infcl_status st, const std::string& msg) {
  set_last_error(msg);
  return st;
}

const char* last_error_string() { return g_last_error.c_str(); }

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

infcl_status make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                            uint32_t box_cols, uint32_t box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return fail(INFCL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(INFCL_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") rows=" +
                                    std::to_string(rows) + " cols=" + std::to_string(cols));
  return INFCL_OK;
}

infcl_status make_tmap_f32_sw128(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                                 uint32_t box_cols, uint32_t box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return fail(INFCL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(INFCL_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (" + std::to_string((int)r) + ")");
  return INFCL_OK;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

static thread_local int g_carve_pairs = 0;
int max_pairs() {
  int pairs = std::max(1, num_sms() / 2 - g_carve_pairs);
  if (const char* e = getenv("INFCL_PAIRS")) pairs = std::max(1, std::min(pairs, atoi(e)));  // diagnostic
  return pairs;
}
PairCarveOut::PairCarveOut(int pairs) : saved(g_carve_pairs) { g_carve_pairs = std::max(0, pairs); }
PairCarveOut::~PairCarveOut() { g_carve_pairs = saved; }

}  // namespace infcl

extern "C" const char* infcl_status_string(infcl_status s) {
  switch (s) {
    case INFCL_OK: return "INFCL_OK";
    case INFCL_ERR_INVALID_ARG: return "INFCL_ERR_INVALID_ARG";
    case INFCL_ERR_SHAPE: return "INFCL_ERR_SHAPE";
    case INFCL_ERR_CONFIG: return "INFCL_ERR_CONFIG";
    case INFCL_ERR_CUDA: return "INFCL_ERR_CUDA";
    case INFCL_ERR_NCCL: return "INFCL_ERR_NCCL";
    case INFCL_ERR_WORKSPACE: return "INFCL_ERR_WORKSPACE";
    case INFCL_ERR_UNSUPPORTED: return "INFCL_ERR_UNSUPPORTED";
  }
  return "INFCL_ERR_UNKNOWN";
}

extern "C" const char* infcl_last_error(void) { return infcl::g_last_error.c_str(); }

extern "C" int infcl_version(void) { return 100; }

extern "C" int infcl_ring_block(int rank, int world, int step) {
  if (world < 1 || rank < 0 || rank >= world || step < 0 || step >= world) return -1;
  return (rank + step) % world;
}
