// C ABI (include/infcl.h): argument validation, workspace layout, and the per-rank ring schedule of
// Alg.1 (forward) and Alg.3 (backward) around the fused pair kernel.
//
// Ring (reading Q13/Q14/Q15): rank r sends to r-1 and receives from r+1, so at 0-based step k it holds
// block (r + k) mod n.  Forward: the text block T travels (prefetched one step ahead on a comm stream,
// double-buffered) together with its column-LSE state, which makes one extra hop home at the end.
// Backward is two symmetric passes: the dI pass keeps I stationary and
// streams (T, c); the dT pass keeps T stationary and streams (I, r).  Gradients therefore never travel.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <functional>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "host_utils.h"
#include "kernels.h"

using namespace infcl;

#define TRY(x)                      \
  do {                              \
    infcl_status _s = (x);          \
    if (_s != INFCL_OK) return _s;  \
  } while (0)

// ------------------------------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
#define LOAD(name) api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name))
      LOAD(GetUniqueId);
      LOAD(CommInitRank);
      LOAD(CommDestroy);
      LOAD(Send);
      LOAD(Recv);
      LOAD(GroupStart);
      LOAD(GroupEnd);
      LOAD(AllReduce);
      LOAD(GetErrorString);
      LOAD(CommGetAsyncError);
#undef LOAD
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
               api.GroupEnd && api.AllReduce;
    }
  }
  return api;
}

#define INFCL_NCCL_TRY(expr)                                                                                  \
  do {                                                                                                        \
    ncclResult_t _r = (expr);                                                                                 \
    if (_r != ncclSuccess)                                                                                    \
      return fail(INFCL_ERR_NCCL, std::string(#expr) + ": " +                                                 \
                                      (nccl().GetErrorString ? nccl().GetErrorString(_r) : std::to_string(_r))); \
  } while (0)
}  // namespace

// Ring transports (infcl.h): INFCL_TRANSPORT_NCCL -- grouped ncclSend/ncclRecv into the caller's workspace;
// INFCL_TRANSPORT_IPC -- one-sided copy-engine writes over CUDA IPC peer mappings (NVLink/NVSwitch P2P on a
// multi-GPU box, same-device mappings when several ranks share one GPU) into a library-owned receive region,
// synchronised by stream memory operations on 32-bit counters (cuStreamWaitValue32 / cuStreamWriteValue32):
// no SM is used by the exchange, so it overlaps the persistent pair kernels, which occupy every SM.
namespace {
// travelling block, column state, LSE vector, and (fused backward ring) the travelling fp32 dT partial of the block
enum XKind { XK_BLK = 0, XK_CS = 1, XK_LSE = 2, XK_DT = 3, XK_N = 4 };

typedef CUresult (*PFN_streamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps {
  PFN_streamValue32 wait = nullptr, write = nullptr;
  bool ok = false;
};
MemOps& memops() {
  static MemOps m;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.wait = reinterpret_cast<PFN_streamValue32>(p);
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.write = reinterpret_cast<PFN_streamValue32>(p);
    m.ok = m.wait && m.write;
  }
  return m;
}

// IPC receive region of one rank (cudaMalloc'ed, exported): a flag page then the receive slots.
struct IpcFlags {
  uint32_t ready[XK_N][2];  // written by rank r+1 after filling slot (kind, s): its fill count
  uint32_t freed[XK_N][2];  // written by rank r-1 after releasing ITS slot (kind, s): its release count
  uint32_t acc_ready[64];   // written by rank q after depositing its loss partial in acc_in[q]: call count
  uint32_t acc_done[64];    // written by rank q after it summed the partials of a call: call count
  double acc_in[64];        // loss partials of every rank (the IPC all-reduce)
  uint32_t hs;              // written by rank r+1 in the connection self-test
  uint32_t hs_data[64];     // copied by rank r+1 in the connection self-test
};
constexpr size_t kFlagBytes = 4096;
static_assert(sizeof(IpcFlags) <= kFlagBytes, "flag page");
}  // namespace (transport)

struct infcl_comm_s {
  int transport = INFCL_TRANSPORT_NCCL;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  cudaStream_t stream = nullptr;  // communication stream (exchange overlapped with compute)
  std::vector<cudaEvent_t> ev;    // event pool
  // NCCL transport: per-call receive slots in the caller's workspace and their arrival events
  void* nslot[XK_N][2] = {};
  cudaEvent_t evr[XK_N][2] = {};
  // IPC transport
  uint8_t* region = nullptr;
  size_t cap[XK_N] = {}, off[XK_N] = {}, region_bytes = 0;
  int64_t max_b = 0;
  int max_d = 0;
  std::vector<uint8_t*> peers;  // mapped receive regions of every rank (peers[rank] = region)
  bool connected = false;
  uint32_t fills[XK_N][2] = {}, rels[XK_N][2] = {}, calls = 0;
  unsigned wait_flags = CU_STREAM_WAIT_VALUE_GEQ;  // | CU_STREAM_WAIT_VALUE_FLUSH where the device supports it
};

namespace {
infcl_status make_comm_stream(infcl_comm c) {
  INFCL_CUDA_TRY(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, -1));
  c->ev.resize(8);
  for (auto& e : c->ev) INFCL_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& row : c->evr)
    for (auto& e : row) INFCL_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return INFCL_OK;
}
}  // namespace

extern "C" infcl_status infcl_get_unique_id(void* id128) {
  if (!id128) return fail(INFCL_ERR_INVALID_ARG, "null id buffer");
  if (!nccl().ok) return fail(INFCL_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  INFCL_NCCL_TRY(nccl().GetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
  return INFCL_OK;
}

extern "C" infcl_status infcl_comm_init(infcl_comm* out, int rank, int world, const void* id128, int device) {
  if (!out || !id128) return fail(INFCL_ERR_INVALID_ARG, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(INFCL_ERR_CONFIG, "rank out of range");
  if (!nccl().ok) return fail(INFCL_ERR_NCCL, "libnccl.so.2 could not be loaded");
  INFCL_CUDA_TRY(cudaSetDevice(device));
  auto* c = new infcl_comm_s();
  c->rank = rank;
  c->world = world;
  c->device = device;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclResult_t r = nccl().CommInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(INFCL_ERR_NCCL, "ncclCommInitRank failed");
  }
  if (infcl_status st = make_comm_stream(c)) {
    infcl_comm_destroy(c);
    return st;
  }
  *out = c;
  return INFCL_OK;
}

extern "C" infcl_status infcl_comm_destroy(infcl_comm c) {
  if (!c) return INFCL_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto e : c->ev) cudaEventDestroy(e);
  for (auto& row : c->evr)
    for (auto e : row)
      if (e) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->comm) nccl().CommDestroy(c->comm);
  for (int q = 0; q < (int)c->peers.size(); ++q)
    if (q != c->rank && c->peers[q]) cudaIpcCloseMemHandle(c->peers[q]);
  if (c->region) cudaFree(c->region);
  delete c;
  return INFCL_OK;
}

// ---- IPC transport setup: create (allocate + zero the receive region), export, connect (map every peer)
extern "C" infcl_status infcl_comm_init_ipc(infcl_comm* out, int rank, int world, int device, int64_t max_b,
                                            int max_d, infcl_dtype dt) {
  if (!out) return fail(INFCL_ERR_INVALID_ARG, "null argument");
  if (world < 2 || world > 64 || rank < 0 || rank >= world)
    return fail(INFCL_ERR_CONFIG, "IPC ring needs 2 <= world <= 64 and 0 <= rank < world");
  if (max_b < world || max_d < 8 || max_b % world) return fail(INFCL_ERR_SHAPE, "bad max_b / max_d");
  if (!memops().ok) return fail(INFCL_ERR_UNSUPPORTED, "cuStreamWaitValue32/cuStreamWriteValue32 unavailable");
  INFCL_CUDA_TRY(cudaSetDevice(device));
  auto* c = new infcl_comm_s();
  c->transport = INFCL_TRANSPORT_IPC;
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->max_b = max_b;
  c->max_d = max_d;
  const size_t bs = (size_t)(max_b / world), dk = dt == INFCL_FP32 ? 3 * (size_t)max_d : (size_t)max_d;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  c->cap[XK_BLK] = al(bs * dk * 2);
  c->cap[XK_CS] = al(bs * sizeof(float2));
  c->cap[XK_LSE] = al(bs * sizeof(float));
  c->cap[XK_DT] = dt == INFCL_BF16 ? al(bs * (size_t)max_d * sizeof(float)) : 0;  // fused backward ring (bf16)
  size_t o = kFlagBytes;
  for (int k = 0; k < XK_N; ++k) {
    c->off[k] = o;
    o += 2 * c->cap[k];
  }
  c->region_bytes = o;
  cudaError_t e = cudaMalloc(&c->region, o);
  if (e != cudaSuccess) {
    delete c;
    return fail(INFCL_ERR_CUDA, std::string("IPC region cudaMalloc: ") + cudaGetErrorString(e));
  }
  if ((e = cudaMemset(c->region, 0, kFlagBytes)) != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) {
    infcl_comm_destroy(c);
    return fail(INFCL_ERR_CUDA, std::string("IPC region init: ") + cudaGetErrorString(e));
  }
  if (infcl_status st = make_comm_stream(c)) {
    infcl_comm_destroy(c);
    return st;
  }
  // peer (NVLink) writes that reached this device before a flag are made visible to the work after the wait
  int can_flush = 0;
  if (cudaDeviceGetAttribute(&can_flush, cudaDevAttrCanFlushRemoteWrites, device) == cudaSuccess && can_flush)
    c->wait_flags |= CU_STREAM_WAIT_VALUE_FLUSH;
  *out = c;
  return INFCL_OK;
}

extern "C" infcl_status infcl_comm_ipc_handle(infcl_comm c, void* handle64) {
  if (!c || !handle64 || c->transport != INFCL_TRANSPORT_IPC) return fail(INFCL_ERR_INVALID_ARG, "not an IPC comm");
  cudaIpcMemHandle_t h;
  INFCL_CUDA_TRY(cudaSetDevice(c->device));
  INFCL_CUDA_TRY(cudaIpcGetMemHandle(&h, c->region));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, sizeof(h));
  return INFCL_OK;
}

extern "C" infcl_status infcl_comm_ipc_connect(infcl_comm c, const void* handles) {
  if (!c || !handles || c->transport != INFCL_TRANSPORT_IPC) return fail(INFCL_ERR_INVALID_ARG, "not an IPC comm");
  if (c->connected) return INFCL_OK;
  INFCL_CUDA_TRY(cudaSetDevice(c->device));
  c->peers.assign(c->world, nullptr);
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) {
      c->peers[q] = c->region;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const uint8_t*>(handles) + 64 * (size_t)q, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(INFCL_ERR_CUDA, "cudaIpcOpenMemHandle(rank " + std::to_string(q) + "): " +
                                                          cudaGetErrorString(e));
    c->peers[q] = static_cast<uint8_t*>(p);
  }
  c->connected = true;
  return INFCL_OK;
}

extern "C" int infcl_comm_transport(infcl_comm c) { return c ? c->transport : -1; }


extern "C" size_t infcl_comm_ipc_region_bytes(infcl_comm c) { return c ? c->region_bytes : 0; }

// ------------------------------------------------------------------------------------------ workspace
namespace {
constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {
  int bs = 0, d = 0, dk = 0, world = 1;
  bool f32 = false;
  PassGeom g{};
  long long slot_ld = 0;
  size_t off_slots, off_rparts, off_rstate, off_cstate, off_own2, off_ring_lse, off_ring_blk, off_ring_dt, off_expA,
      off_expB, off_dscr, off_tails, off_xstate, off_acc, total;
  GcPlan gc{};    // fused single-pass backward (world 1, bf16): its ring shares the forward's column-slot region
  Gc3Plan gc3{};  // three-role variant (d <= 512), preferred when it applies
  size_t gc_bytes() const { return std::max(gc.ok ? gc.bytes : (size_t)0, gc3.ok ? gc3.bytes : (size_t)0); }
};

// ring_ws: the ring's receive buffers live in the workspace (NCCL transport); the IPC transport receives
// into its own exported region, so its workspace has none
Layout make_layout(int64_t b, int d, int world, infcl_dtype dt, bool ring_ws = true) {
  Layout L;
  L.bs = (int)(b / world);
  L.d = d;
  L.world = world;
  L.f32 = dt == INFCL_FP32;
  L.dk = L.f32 ? 3 * d : d;
  L.g = pass_geom(L.bs, L.bs);
  L.slot_ld = (long long)L.g.n_ct * kColsPerTile;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += align_up(bytes);
    return at;
  };
  // column slots (forward) and split-tail scratch (two-pass backward) share one region with the fused
  // backward's step counters and G ring: the three are never live in the same launch
  const size_t slots_b = align_up((size_t)2 * L.g.npairs * L.slot_ld * sizeof(float2));
  // backward: per-pair partials of split tail row blocks (< 2P slots of 128 rows x dk fp32; any row range of the
  // pass has at most P - 1 tail row blocks), combined in pair order -> deterministic gradients
  const size_t tails_b = align_up((size_t)(2 * L.g.npairs - 1) * kRowsPerPair * L.dk * sizeof(float));
  if (!L.f32) {
    L.gc = gc_plan(L.bs, L.bs, L.dk);  // every ring step is a b_s x b_s block
    if (world == 1) L.gc3 = gc3_plan(L.bs, L.bs, L.dk);
  }
  L.off_slots = take(std::max(slots_b + tails_b, L.gc_bytes()));
  L.off_tails = L.off_slots + slots_b;
  // row partials: (row blocks + 2 x pairs) x rows-per-pair slots of whichever kernel runs (narrow or wide)
  const PassGeom gw = wide_geom(L.bs, L.bs);
  L.off_rparts = take(std::max((size_t)(L.g.n_rb + 2 * L.g.npairs) * L.g.rpp,
                               (size_t)(gw.n_rb + 2 * gw.npairs) * gw.rpp) * sizeof(float2));
  L.off_rstate = take((size_t)L.bs * sizeof(float2));
  L.off_cstate = take((size_t)3 * L.bs * sizeof(float2));
  L.off_own2 = take((size_t)2 * L.bs * sizeof(float));
  L.off_ring_lse = take(world > 1 && ring_ws ? (size_t)2 * L.bs * sizeof(float) : 0);
  L.off_ring_blk = take(world > 1 && ring_ws ? (size_t)2 * L.bs * L.dk * 2 : 0);
  // fused backward ring (NCCL transport): receive slots of the travelling dT partial
  L.off_ring_dt = take(world > 1 && ring_ws && L.gc.ok ? (size_t)2 * L.bs * L.d * sizeof(float) : 0);
  L.off_expA = take(L.f32 ? (size_t)L.bs * L.dk * 2 : 0);
  L.off_expB = take(L.f32 ? (size_t)L.bs * L.dk * 2 : 0);
  L.off_dscr = take(L.f32 ? (size_t)L.bs * L.dk * sizeof(float) : 0);
  // NT-Xent (infcl_ntxent_*): the travelling (unused) column state of the self-similarity rings
  L.off_xstate = take((size_t)L.bs * sizeof(float2));
  L.off_acc = take(64);
  L.total = o;
  return L;
}

infcl_status validate(const void* I, const void* T, infcl_dtype dt, int64_t b, int d, float s, int rank, int world,
                      const void* ws, size_t ws_bytes, size_t need) {
  if (!I || !T) return fail(INFCL_ERR_INVALID_ARG, "null feature pointer");
  if (dt != INFCL_BF16 && dt != INFCL_FP32) return fail(INFCL_ERR_INVALID_ARG, "bad dtype");
  if (!std::isfinite(s) || s < 0.f) return fail(INFCL_ERR_INVALID_ARG, "logit scale must be finite and >= 0");
  if (b < 1 || d < 1) return fail(INFCL_ERR_SHAPE, "b and d must be >= 1");
  if (d % 8) return fail(INFCL_ERR_SHAPE, "d must be a multiple of 8 (16-byte TMA rows)");
  if ((dt == INFCL_BF16 && d > kMaxD) || (dt == INFCL_FP32 && 3 * d > kMaxD))
    return fail(INFCL_ERR_SHAPE, "d=" + std::to_string(d) + " above the kernel limit (768 bf16, 256 fp32)");
  if (world < 1 || rank < 0 || rank >= world) return fail(INFCL_ERR_CONFIG, "rank out of range");
  if (b % world)
    return fail(INFCL_ERR_CONFIG, "b=" + std::to_string(b) + " not divisible by world=" + std::to_string(world));
  if (b / world > (int64_t)1 << 30) return fail(INFCL_ERR_SHAPE, "per-rank batch too large");
  if (!ws || ws_bytes < need)
    return fail(INFCL_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  if ((reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return fail(INFCL_ERR_WORKSPACE, "workspace not 256-B aligned");
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(INFCL_ERR_UNSUPPORTED, "no CUDA device");
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) return fail(INFCL_ERR_UNSUPPORTED, "device is not sm_100 (B200)");
  return INFCL_OK;
}

// Per-rank view of the workspace and the rank's operands (expanded to bf16 K-width dk).
struct Rank {
  Layout L;
  uint8_t* ws = nullptr;
  const __nv_bfloat16* A = nullptr;  // image side I (or I' = [hi|hi|lo] for fp32)
  const __nv_bfloat16* B = nullptr;  // text side  T (or T' = [hi|lo|hi])
  const void* I_orig = nullptr;
  const void* T_orig = nullptr;
  float s = 0.f;
  int64_t b = 0;
  float2* slots() const { return reinterpret_cast<float2*>(ws + L.off_slots); }
  float2* rparts() const { return reinterpret_cast<float2*>(ws + L.off_rparts); }
  float2* rstate() const { return reinterpret_cast<float2*>(ws + L.off_rstate); }
  float2* cstate(int i) const { return reinterpret_cast<float2*>(ws + L.off_cstate) + (size_t)i * L.bs; }
  float* own2(int i) const { return reinterpret_cast<float*>(ws + L.off_own2) + (size_t)i * L.bs; }
  float* ring_lse(int i) const { return reinterpret_cast<float*>(ws + L.off_ring_lse) + (size_t)i * L.bs; }
  float* ring_dt(int i) const { return reinterpret_cast<float*>(ws + L.off_ring_dt) + (size_t)i * L.bs * L.d; }
  __nv_bfloat16* ring_blk(int i) const {
    return reinterpret_cast<__nv_bfloat16*>(ws + L.off_ring_blk) + (size_t)i * L.bs * L.dk;
  }
  float* dscr() const { return reinterpret_cast<float*>(ws + L.off_dscr); }
  double* acc() const { return reinterpret_cast<double*>(ws + L.off_acc); }
  float* tails() const { return reinterpret_cast<float*>(ws + L.off_tails); }
  float2* xstate(int i) const { return reinterpret_cast<float2*>(ws + L.off_xstate) + (size_t)i * L.bs; }
};

infcl_status prepare_rank(Rank& R, const void* I, const void* T, infcl_dtype dt, int64_t b, int d, float s, int world,
                          void* ws, cudaStream_t st, bool ring_ws = true) {
  R.L = make_layout(b, d, world, dt, ring_ws);
  R.ws = static_cast<uint8_t*>(ws);
  R.s = s;
  R.b = b;
  R.I_orig = I;
  R.T_orig = T;
  if (dt == INFCL_FP32) {
    auto* eA = reinterpret_cast<__nv_bfloat16*>(R.ws + R.L.off_expA);
    auto* eB = reinterpret_cast<__nv_bfloat16*>(R.ws + R.L.off_expB);
    launch_split_f32(static_cast<const float*>(I), eA, R.L.bs, d, 0, st);
    launch_split_f32(static_cast<const float*>(T), eB, R.L.bs, d, 1, st);
    R.A = eA;
    R.B = eB;
  } else {
    R.A = static_cast<const __nv_bfloat16*>(I);
    R.B = static_cast<const __nv_bfloat16*>(T);
  }
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}

// ---- forward pieces
infcl_status fwd_begin(Rank& R, cudaStream_t st) {
  launch_init_state(R.rstate(), R.L.bs, st);
  launch_init_state(R.cstate(0), R.L.bs, st);
  return INFCL_OK;
}

// main kernel of one ring step: stationary rows A vs held block; then fold row partials
infcl_status fwd_step_main(Rank& R, const __nv_bfloat16* held, bool own, float* diag, cudaStream_t st) {
  PassArgs a{};
  a.A = R.A;
  a.B = held;
  a.nrows = a.ncols = R.L.bs;
  a.dk = a.ld = R.L.dk;
  a.scale = R.s;
  a.diag_on = own ? 1 : 0;
  a.col_slots = R.slots();
  a.slot_ld = R.L.slot_ld;
  a.row_parts = R.rparts();
  a.diag_out = own ? diag : nullptr;
  return launch_pair_forward(a, st);
}

// the step's row partials into the row state and its column slots into the held block's column state
void fwd_step_merge(Rank& R, float2* held_cstate, cudaStream_t st) {
  launch_merge_step(R.rparts(), R.rstate(), R.L.bs, R.slots(), R.L.slot_ld, held_cstate, R.L.bs,
                    fwd_geom(R.L.bs, R.L.bs), st);
}

void fwd_finish(Rank& R, const float2* own_cstate, float* row_lse, float* col_lse, const float* diag, double* acc,
                cudaStream_t st) {
  launch_fwd_finish(R.rstate(), own_cstate, row_lse, col_lse, diag, R.L.bs, acc, st);
}

// ---- backward pieces
infcl_status bwd_step(Rank& R, const __nv_bfloat16* rowsA, const float* lse_rows2, const __nv_bfloat16* held,
                      const float* lse_cols2, bool own, float* dst, int ld_dst, const float* grad, cudaStream_t st,
                      bool self_mask = false) {
  PassArgs a{};
  a.A = rowsA;
  a.B = held;
  a.nrows = a.ncols = R.L.bs;
  a.dk = a.ld = R.L.dk;
  a.scale = R.s;
  a.diag_on = own && !self_mask ? 1 : 0;
  a.self_mask = own && self_mask ? 1 : 0;
  a.lse_row2 = lse_rows2;
  a.lse_col2 = lse_cols2;
  a.dA = dst;
  a.ld_dA = ld_dst;
  a.d_out = R.L.dk;
  a.grad = grad;
  a.coef_base = (float)((double)R.s / (2.0 * (double)R.b));
  a.tail_scratch = R.tails();
  return launch_pair_backward(a, st);
}

// INFCL_FUSED_RING=0 keeps the two-pass backward at world > 1 (INFCL_FUSED_BWD=0 disables every fused path)
bool fused_ring_enabled() {
  static const bool on = [] {
    const char* e = getenv("INFCL_FUSED_RING");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// single-pass backward of the own pair (world 1, bf16): dI (rows I) and dT (columns T) from one fused launch;
// both outputs already hold their exact diagonal terms (diag_init).  INFCL_ERR_UNSUPPORTED = not all CTA pairs
// co-resident (the caller falls back to the two passes)
infcl_status bwd_fused(Rank& R, float* dI, float* dT, const float* grad, cudaStream_t st,
                       const __nv_bfloat16* held = nullptr, const float* held2 = nullptr, bool own = true,
                       bool allow3 = true) {
  PassArgs a{};
  a.A = R.A;
  a.B = held ? held : R.B;
  a.nrows = a.ncols = R.L.bs;
  a.dk = a.ld = R.L.dk;
  a.scale = R.s;
  a.diag_on = own ? 1 : 0;
  a.lse_row2 = R.own2(0);
  a.lse_col2 = held2 ? held2 : R.own2(1);
  a.dA = dI;
  a.ld_dA = R.L.d;
  a.d_out = R.L.dk;
  a.grad = grad;
  a.coef_base = (float)((double)R.s / (2.0 * (double)R.b));
  a.dB = dT;
  a.ld_dB = R.L.d;
  a.gc_ws = R.ws + R.L.off_slots;
  a.gc_ws_bytes = R.L.gc_bytes();
  if (allow3 && R.L.gc3.ok) {
    const infcl_status s3 = launch_bwd3(a, st);
    if (s3 != INFCL_ERR_UNSUPPORTED) return s3;
  }
  return launch_pair_backward_fused(a, st);
}

// ---- blocked single-rank pieces (the host end-to-end entry pipelines PCIe copies against them)
// forward over the block (stationary rows [r0, r1) of I) x (columns [c0, c1) of T) of the own pair: row
// partials merged into rstate right after the launch; column partials accumulate in the (pre-initialised,
// global-column) slots and are merged once by fwd_blocks_finish
void fwd_blocks_begin(Rank& R, cudaStream_t st) {
  launch_init_state(R.slots(), (int)(2LL * R.L.g.npairs * R.L.slot_ld), st);
}
infcl_status fwd_block(Rank& R, int r0, int r1, int c0, int c1, float* diag, cudaStream_t st) {
  PassArgs a{};
  a.A = R.A + (size_t)r0 * R.L.dk;
  a.B = R.B + (size_t)c0 * R.L.dk;
  a.nrows = r1 - r0;
  a.ncols = c1 - c0;
  a.dk = a.ld = R.L.dk;
  a.scale = R.s;
  a.diag_on = std::max(r0, c0) < std::min(r1, c1) ? 1 : 0;
  a.row_off = r0 - c0;
  a.slots_merge = 1;
  a.col_slots = R.slots() + c0;
  a.slot_ld = R.L.slot_ld;
  a.row_parts = R.rparts();
  a.diag_out = diag + r0;
  infcl_status s = launch_pair_forward(a, st);
  if (s) return s;
  launch_merge_rows(R.rparts(), R.rstate() + r0, a.nrows, fwd_geom(a.nrows, a.ncols), st);
  return INFCL_OK;
}
void fwd_blocks_finish(Rank& R, cudaStream_t st) {
  launch_merge_cols(R.slots(), R.L.slot_ld, R.cstate(0), R.L.bs, R.L.g, st, /*all_valid=*/true);
}

// dT pass over stationary rows [r0, r1) of T (own block of I streamed); dT holds its exact diagonal term already
// (diag_init)
infcl_status bwd_dT_chunk(Rank& R, int r0, int r1, const float* grad, float* dT, cudaStream_t st) {
  PassArgs a{};
  a.A = R.B + (size_t)r0 * R.L.dk;
  a.B = R.A;
  a.nrows = r1 - r0;
  a.ncols = R.L.bs;
  a.dk = a.ld = R.L.dk;
  a.scale = R.s;
  a.diag_on = 1;
  a.row_off = r0;
  a.lse_row2 = R.own2(1) + r0;
  a.lse_col2 = R.own2(0);
  a.dA = dT + (size_t)r0 * R.L.d;
  a.ld_dA = R.L.d;
  a.d_out = R.L.dk;
  a.grad = grad;
  a.coef_base = (float)((double)R.s / (2.0 * (double)R.b));
  a.tail_scratch = R.tails();
  infcl_status s = launch_pair_backward(a, st);
  if (s) return s;
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}

// bf16: the pass output starts as its exact fp32 diagonal term (reading H7) and the pair kernel's red.add drains
// accumulate onto it -- one write instead of a memset plus a later read-modify-write.  pass 0 (dI): B_i = T_i;
// pass 1 (dT): B_i = I_i.  fp32 inputs accumulate into the 3d-wide scratch (zeroed) and add the term in pass_end.
void diag_init(Rank& R, int pass, float* out, const float* diag, const float* row_lse, const float* col_lse,
               const float* grad, cudaStream_t st) {
  launch_diag_term(out, R.L.d, pass == 0 ? R.T_orig : R.I_orig, R.L.d, 0, diag, row_lse, col_lse, grad,
                   (float)((double)R.s / (2.0 * (double)R.b)), R.L.bs, R.L.d, /*init=*/true, st);
}

infcl_status bwd_begin(Rank& R, const float* row_lse, const float* col_lse, const float* diag, const float* grad,
                       float* dI, cudaStream_t st) {
  launch_scale_log2(row_lse, R.own2(0), R.L.bs, st);
  launch_scale_log2(col_lse, R.own2(1), R.L.bs, st);
  if (R.L.f32) {
    INFCL_CUDA_TRY(cudaMemsetAsync(R.dscr(), 0, (size_t)R.L.bs * R.L.dk * sizeof(float), st));
  } else {
    diag_init(R, 0, dI, diag, row_lse, col_lse, grad, st);
  }
  return INFCL_OK;
}

// dst of pass 0 (dI) / pass 1 (dT): fp32 mode accumulates into the 3d-wide scratch then combines
float* pass_dst(Rank& R, float* out) { return R.L.f32 ? R.dscr() : out; }

infcl_status pass_end(Rank& R, int pass, float* out, const float* diag, const float* row_lse, const float* col_lse,
                      const float* grad, cudaStream_t st) {
  if (R.L.f32) {  // fp32: combine the hi/lo partials, then add the diagonal term (bf16: diag_init did it)
    launch_combine_f32(R.dscr(), R.L.dk, out, R.L.bs, R.L.d, pass == 0 ? 0 : 1, st);
    const void* Bi = pass == 0 ? R.T_orig : R.I_orig;
    launch_diag_term(out, R.L.d, Bi, R.L.d, 1, diag, row_lse, col_lse, grad,
                     (float)((double)R.s / (2.0 * (double)R.b)), R.L.bs, R.L.d, /*init=*/false, st);
    if (pass == 0) INFCL_CUDA_TRY(cudaMemsetAsync(R.dscr(), 0, (size_t)R.L.bs * R.L.dk * sizeof(float), st));
  }
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}

cudaEvent_t ev(infcl_comm c, int i) { return c->ev[i % c->ev.size()]; }

int prev_rank(int r, int n) { return (r - 1 + n) % n; }
int next_rank(int r, int n) { return (r + 1) % n; }

// ---- ring exchange primitives (both transports); every rank runs the same schedule, so the k-th send of
// (kind, s) by rank r and the k-th fill of r's own slot (kind, s) by rank r+1 pair up.
// slot(kind, s): where the block received in slot s lives (NCCL: the caller's workspace; IPC: own region)
void* xslot(infcl_comm c, int kind, int s) {
  return c->transport == INFCL_TRANSPORT_IPC ? c->region + c->off[kind] + (size_t)s * c->cap[kind] : c->nslot[kind][s];
}
size_t off_ready(int kind, int s) { return offsetof(IpcFlags, ready) + (size_t)(2 * kind + s) * 4; }
size_t off_freed(int kind, int s) { return offsetof(IpcFlags, freed) + (size_t)(2 * kind + s) * 4; }
size_t off_acc_ready(int q) { return offsetof(IpcFlags, acc_ready) + (size_t)q * 4; }
size_t off_acc_done(int q) { return offsetof(IpcFlags, acc_done) + (size_t)q * 4; }
#define INFCL_CU_TRY(expr)                                                                              \
  do {                                                                                                  \
    CUresult _r = (expr);                                                                               \
    if (_r != CUDA_SUCCESS) return fail(INFCL_ERR_CUDA, std::string(#expr) + ": CUresult " + std::to_string((int)_r)); \
  } while (0)
// wait on `stream` until the local flag reaches v / write v to a flag of `region` (fenced: earlier work of the
// stream, including copies, is visible before the flag)
infcl_status flag_wait(infcl_comm c, cudaStream_t stream, size_t field, uint32_t v) {
  INFCL_CU_TRY(memops().wait((CUstream)stream, reinterpret_cast<CUdeviceptr>(c->region + field), v, c->wait_flags));
  return INFCL_OK;
}
infcl_status flag_write(cudaStream_t stream, uint8_t* region, size_t field, uint32_t v) {
  INFCL_CU_TRY(memops().write((CUstream)stream, reinterpret_cast<CUdeviceptr>(region + field), v,
                              CU_STREAM_WRITE_VALUE_DEFAULT));
  return INFCL_OK;
}

// device-to-device copy of one travelling block (or state) into the peer's mapped region: one cudaMemcpyAsync
// per message (peer-to-peer across GPUs runs on the copy engines; the batched-copy API is not used because it
// raised GPU faults on this pool)
cudaError_t ce_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st);
}

// send `bytes` of `src` to slot (kind, s) of rank r-1, and (NCCL) receive rank r+1's into our slot (kind, s);
// on the comm stream
infcl_status xsend(infcl_comm c, int kind, int s, const void* src, size_t bytes) {
  const int n = c->world, r = c->rank;
  if (c->transport == INFCL_TRANSPORT_NCCL) {
    INFCL_NCCL_TRY(nccl().GroupStart());
    INFCL_NCCL_TRY(nccl().Send(src, bytes, ncclUint8, prev_rank(r, n), c->comm, c->stream));
    INFCL_NCCL_TRY(nccl().Recv(c->nslot[kind][s], bytes, ncclUint8, next_rank(r, n), c->comm, c->stream));
    INFCL_NCCL_TRY(nccl().GroupEnd());
    INFCL_CUDA_TRY(cudaEventRecord(c->evr[kind][s], c->stream));
    return INFCL_OK;
  }
  if (bytes > c->cap[kind]) return fail(INFCL_ERR_WORKSPACE, "message larger than the IPC region slot");
  // the previous fills of rank r-1's slot (kind, s) must all have been released by r-1
  TRY(flag_wait(c, c->stream, off_freed(kind, s), c->fills[kind][s]));
  uint8_t* dst = c->peers[prev_rank(r, n)] + c->off[kind] + (size_t)s * c->cap[kind];
  INFCL_CUDA_TRY(ce_copy(dst, src, bytes, c->stream));
  ++c->fills[kind][s];
  return flag_write(c->stream, c->peers[prev_rank(r, n)], off_ready(kind, s), c->fills[kind][s]);
}
// make `stream` wait until our slot (kind, s) holds the fill that pairs with our latest xsend(kind, s)
infcl_status xwait(infcl_comm c, cudaStream_t stream, int kind, int s) {
  if (c->transport == INFCL_TRANSPORT_NCCL) {
    INFCL_CUDA_TRY(cudaStreamWaitEvent(stream, c->evr[kind][s], 0));
    return INFCL_OK;
  }
  return flag_wait(c, stream, off_ready(kind, s), c->fills[kind][s]);
}
// our slot (kind, s) is no longer read (ordered on `stream`): rank r+1 may refill it
infcl_status xrelease(infcl_comm c, cudaStream_t stream, int kind, int s) {
  if (c->transport == INFCL_TRANSPORT_NCCL) return INFCL_OK;
  ++c->rels[kind][s];
  return flag_write(stream, c->peers[next_rank(c->rank, c->world)], off_freed(kind, s), c->rels[kind][s]);
}
// sum of one fp64 per rank into `acc` on every rank, in rank order (deterministic); on the comm stream
infcl_status allreduce_acc(infcl_comm c, double* acc) {
  if (c->transport == INFCL_TRANSPORT_NCCL) {
    INFCL_NCCL_TRY(nccl().AllReduce(acc, acc, 1, ncclFloat64, ncclSum, c->comm, c->stream));
    return INFCL_OK;
  }
  const int n = c->world, r = c->rank;
  const uint32_t call = ++c->calls;
  for (int q = 0; q < n; ++q) {  // deposit our partial in acc_in[r] of every rank (q == r: our own region)
    if (q != r) TRY(flag_wait(c, c->stream, off_acc_done(q), call - 1));  // q summed the last call
    INFCL_CUDA_TRY(ce_copy(c->peers[q] + offsetof(IpcFlags, acc_in) + r * sizeof(double), acc, sizeof(double),
                           c->stream));
    if (q != r) TRY(flag_write(c->stream, c->peers[q], off_acc_ready(r), call));
  }
  for (int q = 0; q < n; ++q)
    if (q != r) TRY(flag_wait(c, c->stream, off_acc_ready(q), call));
  launch_sum_f64(reinterpret_cast<const double*>(c->region + offsetof(IpcFlags, acc_in)), n, acc, c->stream);
  for (int q = 0; q < n; ++q)
    if (q != r) TRY(flag_write(c->stream, c->peers[q], off_acc_done(r), call));
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}
// non-blocking check for an asynchronous NCCL failure on the ring (a peer died, a network error): reported as
// INFCL_ERR_NCCL instead of surfacing later as a hang
infcl_status comm_async_check(infcl_comm c) {
  if (!c || !c->comm || !nccl().CommGetAsyncError) return INFCL_OK;
  ncclResult_t r = ncclSuccess;
  if (nccl().CommGetAsyncError(c->comm, &r) != ncclSuccess || (r != ncclSuccess && r != ncclInProgress))
    return fail(INFCL_ERR_NCCL, std::string("asynchronous NCCL error: ") +
                                    (nccl().GetErrorString ? nccl().GetErrorString(r) : std::to_string(r)));
  return INFCL_OK;
}
}  // namespace

namespace {
// ---- the ring schedule as data (Alg.1 forward, Alg.3 backward passes; readings Q13-Q15).  One generator
// emits the per-rank op list; the executor below runs it with either transport, and infcl_ring_schedule
// exports it so tests/test_ring_schedule.py can check it on the CPU: random interleavings of n ranks' two
// streams under both transports' semantics must never read a slot before its fill, overwrite a slot that is
// still to be read, or deadlock.
enum RingOp : int32_t {
  OP_EVREC = 1,   // a = stream, b = event
  OP_EVWAIT = 2,  // a = stream, b = event
  OP_SEND = 3,    // on comm: a = kind, b = slot, c = source buffer, tag = block id carried
  OP_WAITV = 4,   // a = stream, b = kind, c = slot: the slot's pairing fill has landed
  OP_RELEASE = 5, // a = stream, b = kind, c = slot: the slot may be refilled
  OP_COMPUTE = 6, // on st: a = block buffer, b = LSE buffer (backward) or -9, c = step k, tag = block id
  OP_MERGE = 7,   // on st (forward): a = column-state buffer (read-modify-write), tag = its block id
  OP_FINISH = 8,  // on st (forward): a = column-state buffer, tag = own block id
  OP_ALLRED = 9   // the loss all-reduce (comm stream, collective)
};
enum RingStream : int32_t { RS_ST = 0, RS_COMM = 1 };
// buffer references: >= 0 a receive slot 2*kind + s; BUF_OWN the pass's own travelling block (T forward /
// dI pass, I in the dT pass), BUF_OWNL its own LSE vector, BUF_OWNCS the own initial column state
constexpr int32_t BUF_OWN = -1, BUF_OWNL = -2, BUF_OWNCS = -3, BUF_NONE = -9;
struct ROp {
  int32_t code, a, b, c, tag;
};
inline int32_t slot_ref(int kind, int s) { return 2 * kind + s; }

void fwd_ring_ops(int n, int r, std::vector<ROp>& o) {
  o.push_back({OP_EVREC, RS_ST, 0, 0, -1});
  o.push_back({OP_EVWAIT, RS_COMM, 0, 0, -1});  // inputs ready before the first send
  int32_t held = BUF_OWN;
  for (int k = 0; k < n; ++k) {
    const int32_t blk = (r + k) % n;  // block held at step k (reading Q13)
    if (k + 1 < n) {
      // forwarding a received block: the comm stream itself must see it arrive (IPC: the fill is a remote
      // write, not ordered on this stream)
      if (k >= 1) o.push_back({OP_WAITV, RS_COMM, XK_BLK, (k - 1) & 1, -1});
      o.push_back({OP_SEND, XK_BLK, k & 1, held, blk});  // prefetch the block held at step k+1
      o.push_back({OP_EVREC, RS_COMM, 2, 0, -1});
    }
    o.push_back({OP_COMPUTE, held, BUF_NONE, k, blk});
    const int32_t cs = k == 0 ? BUF_OWNCS : slot_ref(XK_CS, (k - 1) & 1);
    if (k >= 1) o.push_back({OP_WAITV, RS_ST, XK_CS, (k - 1) & 1, -1});  // held block's column state arrived
    o.push_back({OP_MERGE, cs, 0, 0, blk});
    o.push_back({OP_EVREC, RS_ST, 1, 0, -1});  // compute of step k done
    o.push_back({OP_EVWAIT, RS_COMM, 1, 0, -1});
    o.push_back({OP_SEND, XK_CS, k & 1, cs, blk});  // column state onward (last: the hop home)
    if (k >= 1) o.push_back({OP_RELEASE, RS_COMM, XK_CS, (k - 1) & 1, -1});
    if (k + 1 < n) {
      o.push_back({OP_EVWAIT, RS_ST, 2, 0, -1});  // our forward of `held` is done
      o.push_back({OP_WAITV, RS_ST, XK_BLK, k & 1, -1});  // next block arrived
    }
    if (k >= 1) o.push_back({OP_RELEASE, RS_ST, XK_BLK, (k - 1) & 1, -1});  // computed and forwarded `held`
    held = slot_ref(XK_BLK, k & 1);
  }
  o.push_back({OP_WAITV, RS_ST, XK_CS, (n - 1) & 1, -1});  // own column state is home
  o.push_back({OP_FINISH, slot_ref(XK_CS, (n - 1) & 1), 0, 0, r});
  o.push_back({OP_RELEASE, RS_ST, XK_CS, (n - 1) & 1, -1});
  o.push_back({OP_EVREC, RS_ST, 4, 0, -1});
  o.push_back({OP_EVWAIT, RS_COMM, 4, 0, -1});
  o.push_back({OP_ALLRED, 0, 0, 0, -1});
  o.push_back({OP_EVREC, RS_COMM, 7, 0, -1});
  o.push_back({OP_EVWAIT, RS_ST, 7, 0, -1});
}

// one backward pass (dI pass: rows I, streamed (T, c); dT pass: rows T, streamed (I, r)); gradients never travel
void bwd_ring_ops(int n, int r, std::vector<ROp>& o) {
  o.push_back({OP_EVREC, RS_ST, 0, 0, -1});
  o.push_back({OP_EVWAIT, RS_COMM, 0, 0, -1});
  int32_t held = BUF_OWN, held2 = BUF_OWNL;
  for (int k = 0; k < n; ++k) {
    const int32_t blk = (r + k) % n;
    if (k + 1 < n) {
      if (k >= 1) {
        // (NCCL) our slot k&1 was held at step k-1: its compute must be done before the receive
        o.push_back({OP_EVWAIT, RS_COMM, 5 + ((k - 1) & 1), 0, -1});
        // forwarding received slots: the comm stream must see them arrive
        o.push_back({OP_WAITV, RS_COMM, XK_BLK, (k - 1) & 1, -1});
        o.push_back({OP_WAITV, RS_COMM, XK_LSE, (k - 1) & 1, -1});
      }
      o.push_back({OP_SEND, XK_BLK, k & 1, held, blk});
      o.push_back({OP_SEND, XK_LSE, k & 1, held2, blk});
      o.push_back({OP_EVREC, RS_COMM, 2, 0, -1});
    }
    o.push_back({OP_COMPUTE, held, held2, k, blk});
    o.push_back({OP_EVREC, RS_ST, 5 + (k & 1), 0, -1});
    if (k + 1 < n) {
      o.push_back({OP_EVWAIT, RS_ST, 2, 0, -1});  // our forward of (held, held2) is done
      o.push_back({OP_WAITV, RS_ST, XK_BLK, k & 1, -1});
      o.push_back({OP_WAITV, RS_ST, XK_LSE, k & 1, -1});
    }
    if (k >= 1) {  // computed and forwarded (held, held2): rank r+1 may refill those slots
      o.push_back({OP_RELEASE, RS_ST, XK_BLK, (k - 1) & 1, -1});
      o.push_back({OP_RELEASE, RS_ST, XK_LSE, (k - 1) & 1, -1});
    }
    held = slot_ref(XK_BLK, k & 1);
    held2 = slot_ref(XK_LSE, k & 1);
  }
}

// the fused single-pass backward ring (Alg.3 P:539-558 with the dT partials rotating, as the forward's column
// state does): at step k rank r holds block (T, c) of rank (r + k) mod n and that block's dT partial; the fused
// launch adds this rank's dI rows and the block's dT partial (COMPUTE marks the block / LSE reads, MERGE the
// read-modify-write of the partial, where the launch happens); the partial then moves on to rank r-1, and after
// n steps it is back home complete (the n-th send is the hop home, reading Q15) -> FINISH copies it into dT
void bwd_fused_ring_ops(int n, int r, std::vector<ROp>& o) {
  o.push_back({OP_EVREC, RS_ST, 0, 0, -1});
  o.push_back({OP_EVWAIT, RS_COMM, 0, 0, -1});
  int32_t held = BUF_OWN, held2 = BUF_OWNL;
  for (int k = 0; k < n; ++k) {
    const int32_t blk = (r + k) % n;
    if (k + 1 < n) {
      if (k >= 1) {
        o.push_back({OP_EVWAIT, RS_COMM, 5 + ((k - 1) & 1), 0, -1});
        o.push_back({OP_WAITV, RS_COMM, XK_BLK, (k - 1) & 1, -1});
        o.push_back({OP_WAITV, RS_COMM, XK_LSE, (k - 1) & 1, -1});
      }
      o.push_back({OP_SEND, XK_BLK, k & 1, held, blk});
      o.push_back({OP_SEND, XK_LSE, k & 1, held2, blk});
      o.push_back({OP_EVREC, RS_COMM, 2, 0, -1});
    }
    o.push_back({OP_COMPUTE, held, held2, k, blk});
    const int32_t part = k == 0 ? BUF_OWNCS : slot_ref(XK_DT, (k - 1) & 1);
    if (k >= 1) o.push_back({OP_WAITV, RS_ST, XK_DT, (k - 1) & 1, -1});  // the held block's partial arrived
    o.push_back({OP_MERGE, part, 0, 0, blk});                           // the fused launch
    o.push_back({OP_EVREC, RS_ST, 5 + (k & 1), 0, -1});
    o.push_back({OP_EVREC, RS_ST, 1, 0, -1});
    o.push_back({OP_EVWAIT, RS_COMM, 1, 0, -1});
    o.push_back({OP_SEND, XK_DT, k & 1, part, blk});  // partial onward (last: the hop home)
    if (k >= 1) o.push_back({OP_RELEASE, RS_COMM, XK_DT, (k - 1) & 1, -1});
    if (k + 1 < n) {
      o.push_back({OP_EVWAIT, RS_ST, 2, 0, -1});
      o.push_back({OP_WAITV, RS_ST, XK_BLK, k & 1, -1});
      o.push_back({OP_WAITV, RS_ST, XK_LSE, k & 1, -1});
    }
    if (k >= 1) {
      o.push_back({OP_RELEASE, RS_ST, XK_BLK, (k - 1) & 1, -1});
      o.push_back({OP_RELEASE, RS_ST, XK_LSE, (k - 1) & 1, -1});
    }
    held = slot_ref(XK_BLK, k & 1);
    held2 = slot_ref(XK_LSE, k & 1);
  }
  o.push_back({OP_EVREC, RS_COMM, 3, 0, -1});  // every send (incl. the step-0 send of the own buffer) done
  o.push_back({OP_EVWAIT, RS_ST, 3, 0, -1});
  o.push_back({OP_WAITV, RS_ST, XK_DT, (n - 1) & 1, -1});  // own dT is home
  o.push_back({OP_FINISH, slot_ref(XK_DT, (n - 1) & 1), 0, 0, r});
  o.push_back({OP_RELEASE, RS_ST, XK_DT, (n - 1) & 1, -1});
}

// executor of a ring op list on `st` (compute) and comm's stream, with comm's transport
struct RingCtx {
  const void* own = nullptr;   // BUF_OWN
  const void* ownl = nullptr;  // BUF_OWNL
  float2* owncs = nullptr;     // BUF_OWNCS (forward)
  void* ownpart = nullptr;     // BUF_OWNCS (fused backward ring: the own dT buffer, the step-0 partial)
  size_t bytes[XK_N] = {};
  std::function<infcl_status(int k, const void* blk, const void* lse)> compute;
  std::function<void(float2* cs)> merge;
  std::function<void(const float2* cs)> finish;
  std::function<infcl_status(void* part)> merge_part;  // fused backward ring: the launch on the held partial
  std::function<void(const void* part)> finish_part;
  double* acc = nullptr;
};
infcl_status run_ring(infcl_comm c, const std::vector<ROp>& ops, RingCtx& x, cudaStream_t st) {
  auto ptr = [&](int32_t ref) -> void* {
    if (ref == BUF_OWN) return const_cast<void*>(x.own);
    if (ref == BUF_OWNL) return const_cast<void*>(x.ownl);
    if (ref == BUF_OWNCS) return x.ownpart ? x.ownpart : static_cast<void*>(x.owncs);
    return ref >= 0 ? xslot(c, ref / 2, ref % 2) : nullptr;
  };
  auto strm = [&](int32_t id) { return id == RS_ST ? st : c->stream; };
  for (const ROp& op : ops) {
    switch (op.code) {
      case OP_EVREC: INFCL_CUDA_TRY(cudaEventRecord(ev(c, op.b), strm(op.a))); break;
      case OP_EVWAIT: INFCL_CUDA_TRY(cudaStreamWaitEvent(strm(op.a), ev(c, op.b), 0)); break;
      case OP_SEND: {  // block hops are timed on the comm stream when profiling (infcl_profile_read kind 2)
        cudaEvent_t e0 = op.a == XK_BLK ? profile_begin(c->stream) : nullptr;
        TRY(xsend(c, op.a, op.b, ptr(op.c), x.bytes[op.a]));
        profile_end(2, e0, c->stream);
        break;
      }
      case OP_WAITV: TRY(xwait(c, strm(op.a), op.b, op.c)); break;
      case OP_RELEASE: TRY(xrelease(c, strm(op.a), op.b, op.c)); break;
      case OP_COMPUTE: TRY(x.compute(op.c, ptr(op.a), op.b == BUF_NONE ? nullptr : ptr(op.b))); break;
      case OP_MERGE:
        if (x.merge_part) TRY(x.merge_part(ptr(op.a)));
        else x.merge(static_cast<float2*>(ptr(op.a)));
        break;
      case OP_FINISH:
        if (x.finish_part) x.finish_part(ptr(op.a));
        else x.finish(static_cast<const float2*>(ptr(op.a)));
        break;
      case OP_ALLRED:
        if (x.acc) TRY(allreduce_acc(c, x.acc));  // NT-Xent's self-similarity rings reduce nothing
        break;
      default: return fail(INFCL_ERR_INVALID_ARG, "bad ring op");
    }
  }
  return INFCL_OK;
}

}  // namespace

// The per-rank ring schedule as int32 records of 6 (code, a, b, c, tag, 0); which = 0 forward, 1 backward pass.
// Returns the number of records (or -1 on bad arguments; records beyond `cap` are counted, not written).
extern "C" int infcl_ring_schedule(int world, int rank, int which, int32_t* out, int cap) {
  if (world < 2 || world > 64 || rank < 0 || rank >= world || which < 0 || which > 2) return -1;
  std::vector<ROp> ops;
  if (which == 0) fwd_ring_ops(world, rank, ops);
  else if (which == 1) bwd_ring_ops(world, rank, ops);
  else bwd_fused_ring_ops(world, rank, ops);
  for (int i = 0; i < (int)ops.size() && i < cap && out; ++i) {
    const int32_t rec[6] = {ops[i].code, ops[i].a, ops[i].b, ops[i].c, ops[i].tag, 0};
    std::memcpy(out + 6 * (size_t)i, rec, sizeof(rec));
  }
  return (int)ops.size();
}

// Connection self-test (collective): every rank copies 256 B into rank r-1's region with the transport's own
// copy path, bumps r-1's handshake counter with cuStreamWriteValue32, and waits for its own counter with
// cuStreamWaitValue32 -- the three mechanisms of the ring -- then checks the copied bytes.  A peer path that
// fails returns an error instead of hanging a later call: the host polls for `timeout_ms` and, on timeout,
// releases the stream's wait by writing the counter itself.
extern "C" infcl_status infcl_comm_ipc_selftest(infcl_comm c, int timeout_ms) {
  if (!c || c->transport != INFCL_TRANSPORT_IPC || !c->connected)
    return fail(INFCL_ERR_INVALID_ARG, "not a connected IPC comm");
  INFCL_CUDA_TRY(cudaSetDevice(c->device));
  const int n = c->world, r = c->rank;
  uint32_t pattern[64];
  for (int i = 0; i < 64; ++i) pattern[i] = 0x9E3779B9u * (uint32_t)(r + 1) + (uint32_t)i;
  uint8_t* src = c->region + c->off[XK_LSE];  // own scratch: slot memory is free outside calls
  INFCL_CUDA_TRY(cudaMemcpy(src, pattern, sizeof(pattern), cudaMemcpyHostToDevice));
  INFCL_CUDA_TRY(ce_copy(c->peers[prev_rank(r, n)] + offsetof(IpcFlags, hs_data), src, sizeof(pattern), c->stream));
  TRY(flag_write(c->stream, c->peers[prev_rank(r, n)], offsetof(IpcFlags, hs), 1));
  TRY(flag_wait(c, c->stream, offsetof(IpcFlags, hs), 1));
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t q;
  while ((q = cudaStreamQuery(c->stream)) == cudaErrorNotReady) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms)) {
      const uint32_t one = 1;  // unblock our own stream, then report
      cudaMemcpy(c->region + offsetof(IpcFlags, hs), &one, sizeof(one), cudaMemcpyHostToDevice);
      cudaStreamSynchronize(c->stream);
      return fail(INFCL_ERR_CUDA, "IPC self-test timed out: rank " + std::to_string(next_rank(r, n)) +
                                      " never signalled over its peer mapping");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  if (q != cudaSuccess) return fail(INFCL_ERR_CUDA, std::string("IPC self-test: ") + cudaGetErrorString(q));
  uint32_t got[64];
  INFCL_CUDA_TRY(cudaMemcpy(got, c->region + offsetof(IpcFlags, hs_data), sizeof(got), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 64; ++i)
    if (got[i] != 0x9E3779B9u * (uint32_t)(next_rank(r, n) + 1) + (uint32_t)i)
      return fail(INFCL_ERR_CUDA, "IPC self-test: data from rank " + std::to_string(next_rank(r, n)) + " corrupted");
  return INFCL_OK;
}

extern "C" size_t infcl_workspace_bytes(int64_t b, int d, int world, infcl_dtype dt) {
  if (b < 1 || d < 1 || world < 1 || b % world) return 0;
  return make_layout(b, d, world, dt).total;
}

extern "C" size_t infcl_comm_workspace_bytes(infcl_comm comm, int64_t b, int d, int world, infcl_dtype dt) {
  if (b < 1 || d < 1 || world < 1 || b % world) return 0;
  return make_layout(b, d, world, dt, !(comm && comm->transport == INFCL_TRANSPORT_IPC)).total;
}

namespace {
// checks shared by the ring entry points; binds the NCCL transport's receive slots to this call's workspace
infcl_status ring_setup(infcl_comm comm, const Rank& R, int rank, int world) {
  if (!comm || comm->world != world || comm->rank != rank)
    return fail(INFCL_ERR_CONFIG, "world > 1 needs a communicator with matching rank/world");
  if (comm->transport == INFCL_TRANSPORT_IPC) {
    if (!comm->connected) return fail(INFCL_ERR_CONFIG, "IPC communicator not connected (infcl_comm_ipc_connect)");
    // every message of the schedule must fit its slot BEFORE anything is enqueued: a failing xsend part-way
    // through would leave the fill/release counters of the ring out of step (the next call would wait forever)
    if ((size_t)R.L.bs * R.L.dk * 2 > comm->cap[XK_BLK] || (size_t)R.L.bs * sizeof(float2) > comm->cap[XK_CS] ||
        (size_t)R.L.bs * sizeof(float) > comm->cap[XK_LSE] || (int64_t)R.L.bs > comm->max_b / world ||
        (R.L.gc.ok && (size_t)R.L.bs * R.L.d * sizeof(float) > comm->cap[XK_DT]))
      return fail(INFCL_ERR_WORKSPACE, "shard larger than the IPC region was sized for (max_b, max_d)");
    int dev = -1;
    INFCL_CUDA_TRY(cudaGetDevice(&dev));
    if (dev != comm->device) return fail(INFCL_ERR_CONFIG, "current device differs from the communicator's");
  } else {
    for (int s = 0; s < 2; ++s) {
      comm->nslot[XK_BLK][s] = R.ring_blk(s);
      comm->nslot[XK_CS][s] = R.cstate(1 + s);
      comm->nslot[XK_LSE][s] = R.ring_lse(s);
      comm->nslot[XK_DT][s] = R.L.gc.ok ? R.ring_dt(s) : nullptr;
    }
  }
  return INFCL_OK;
}
bool ring_in_ws(infcl_comm comm) { return !(comm && comm->transport == INFCL_TRANSPORT_IPC); }
// SM carve-out of a ring call: the NCCL transport's send/recv kernels need SMs, and the persistent pair kernels
// hold every SM (one 320-thread CTA with ~200 KB of smem per SM), so with NCCL at world > 1 the pair kernels leave
// INFCL_NCCL_CARVEOUT_PAIRS CTA pairs (default 2 = 4 SMs) free for the exchange to run beside the ring step's
// kernel (survey H6; the P:216-219 overlap).  The IPC transport copies on the copy engines and needs none.
int ring_carveout(infcl_comm comm, int world) {
  if (world <= 1 || !comm || comm->transport != INFCL_TRANSPORT_NCCL) return 0;
  static const int k = [] {
    const char* e = getenv("INFCL_NCCL_CARVEOUT_PAIRS");
    return e ? std::max(0, atoi(e)) : 2;
  }();
  return k;
}
}  // namespace


extern "C" infcl_status infcl_forward(infcl_comm comm, const void* I_local, const void* T_local, infcl_dtype dt,
                                      int64_t b, int d, float s, int rank, int world, float* row_lse, float* col_lse,
                                      float* diag, float* loss, void* ws, size_t ws_bytes, void* stream) {
  const size_t need = infcl_comm_workspace_bytes(world > 1 ? comm : nullptr, b, d, world, dt);
  TRY(validate(I_local, T_local, dt, b, d, s, rank, world, ws, ws_bytes, need));
  if (!row_lse || !col_lse || !diag || !loss) return fail(INFCL_ERR_INVALID_ARG, "null output pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PairCarveOut carve(ring_carveout(comm, world));  // layout and launches of this call see the same pair count
  Rank R;
  TRY(prepare_rank(R, I_local, T_local, dt, b, d, s, world, ws, st, world == 1 || ring_in_ws(comm)));
  if (world > 1) TRY(ring_setup(comm, R, rank, world));
  INFCL_CUDA_TRY(cudaMemsetAsync(R.acc(), 0, sizeof(double), st));
  TRY(fwd_begin(R, st));
  if (world == 1) {
    TRY(fwd_step_main(R, R.B, true, diag, st));
    fwd_step_merge(R, R.cstate(0), st);
    fwd_finish(R, R.cstate(0), row_lse, col_lse, diag, R.acc(), st);
    launch_loss_write(R.acc(), loss, b, st);
    INFCL_CUDA_TRY(cudaGetLastError());
    return INFCL_OK;
  }
  // ---- ring over `world` GPUs (Alg.1): the schedule of fwd_ring_ops, executed with comm's transport
  std::vector<ROp> ops;
  fwd_ring_ops(world, rank, ops);
  RingCtx x;
  x.own = R.B;
  x.owncs = R.cstate(0);
  x.bytes[XK_BLK] = (size_t)R.L.bs * R.L.dk * 2;
  x.bytes[XK_CS] = (size_t)R.L.bs * sizeof(float2);
  x.acc = R.acc();
  x.compute = [&](int k, const void* blk, const void*) {
    return fwd_step_main(R, static_cast<const __nv_bfloat16*>(blk), k == 0, diag, st);
  };
  x.merge = [&](float2* cs) { fwd_step_merge(R, cs, st); };
  x.finish = [&](const float2* cs) { fwd_finish(R, cs, row_lse, col_lse, diag, R.acc(), st); };
  TRY(run_ring(comm, ops, x, st));
  launch_loss_write(R.acc(), loss, b, st);
  TRY(comm_async_check(comm));
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}

static infcl_status backward_impl(infcl_comm comm, const void* I_local, const void* T_local, infcl_dtype dt,
                                  int64_t b, int d, float s, int rank, int world, const float* row_lse,
                                  const float* col_lse, const float* diag, const float* grad, float* dI, float* dT,
                                  void* ws, size_t ws_bytes, void* stream, cudaEvent_t dI_ready) {
  const size_t need = infcl_comm_workspace_bytes(world > 1 ? comm : nullptr, b, d, world, dt);
  TRY(validate(I_local, T_local, dt, b, d, s, rank, world, ws, ws_bytes, need));
  if (!row_lse || !col_lse || !diag || !grad || !dI || !dT) return fail(INFCL_ERR_INVALID_ARG, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PairCarveOut carve(ring_carveout(comm, world));
  Rank R;
  TRY(prepare_rank(R, I_local, T_local, dt, b, d, s, world, ws, st, world == 1 || ring_in_ws(comm)));
  if (world > 1) TRY(ring_setup(comm, R, rank, world));
  TRY(bwd_begin(R, row_lse, col_lse, diag, grad, dI, st));
  if (world == 1 && (R.L.gc.ok || R.L.gc3.ok)) {
    diag_init(R, 1, dT, diag, row_lse, col_lse, grad, st);
    const infcl_status fs = bwd_fused(R, dI, dT, grad, st);
    if (fs == INFCL_OK) {
      if (dI_ready) INFCL_CUDA_TRY(cudaEventRecord(dI_ready, st));
      INFCL_CUDA_TRY(cudaGetLastError());
      return INFCL_OK;
    }
    if (fs != INFCL_ERR_UNSUPPORTED) return fs;
    diag_init(R, 0, dI, diag, row_lse, col_lse, grad, st);  // nothing ran: the two passes start over
  }
  const size_t blk_bytes = (size_t)R.L.bs * R.L.dk * 2, lse_bytes = (size_t)R.L.bs * sizeof(float);
  if (world > 1 && R.L.gc.ok && fused_ring_enabled()) {
    // single pass over the ring: dI stays, the blocks' dT partials rotate (bwd_fused_ring_ops)
    diag_init(R, 1, dT, diag, row_lse, col_lse, grad, st);
    std::vector<ROp> ops;
    bwd_fused_ring_ops(world, rank, ops);
    RingCtx x;
    x.own = R.B;
    x.ownl = R.own2(1);
    x.ownpart = dT;
    x.bytes[XK_BLK] = blk_bytes;
    x.bytes[XK_LSE] = lse_bytes;
    x.bytes[XK_DT] = (size_t)R.L.bs * R.L.d * sizeof(float);
    const __nv_bfloat16* cur_blk = nullptr;
    const float* cur_lse = nullptr;
    int cur_k = 0;
    x.compute = [&](int k, const void* blk, const void* lse) {  // the launch happens at the partial's MERGE
      cur_blk = static_cast<const __nv_bfloat16*>(blk);
      cur_lse = static_cast<const float*>(lse);
      cur_k = k;
      return INFCL_OK;
    };
    x.merge_part = [&](void* part) {
      return bwd_fused(R, dI, static_cast<float*>(part), grad, st, cur_blk, cur_lse, cur_k == 0, false);
    };
    x.finish_part = [&](const void* part) {
      cudaMemcpyAsync(dT, part, x.bytes[XK_DT], cudaMemcpyDeviceToDevice, st);
    };
    TRY(run_ring(comm, ops, x, st));
    if (dI_ready) INFCL_CUDA_TRY(cudaEventRecord(dI_ready, st));
    TRY(comm_async_check(comm));
    INFCL_CUDA_TRY(cudaGetLastError());
    return INFCL_OK;
  }
  for (int pass = 0; pass < 2; ++pass) {
    // pass 0: rows I (lse r), stream (T, c) -> dI;  pass 1: rows T (lse c), stream (I, r) -> dT
    const __nv_bfloat16* rows = pass == 0 ? R.A : R.B;
    const __nv_bfloat16* own_blk = pass == 0 ? R.B : R.A;
    const float* rows2 = R.own2(pass == 0 ? 0 : 1);
    const float* own_cols2 = R.own2(pass == 0 ? 1 : 0);
    float* out = pass == 0 ? dI : dT;
    float* dst = pass_dst(R, out);
    const int ld_dst = R.L.f32 ? R.L.dk : R.L.d;
    if (!R.L.f32 && pass == 1) diag_init(R, 1, dT, diag, row_lse, col_lse, grad, st);
    if (world == 1) {
      TRY(bwd_step(R, rows, rows2, own_blk, own_cols2, true, dst, ld_dst, grad, st));
    } else {
      std::vector<ROp> ops;
      bwd_ring_ops(world, rank, ops);
      RingCtx x;
      x.own = own_blk;
      x.ownl = own_cols2;
      x.bytes[XK_BLK] = blk_bytes;
      x.bytes[XK_LSE] = lse_bytes;
      x.compute = [&](int k, const void* blk, const void* lse) {
        return bwd_step(R, rows, rows2, static_cast<const __nv_bfloat16*>(blk), static_cast<const float*>(lse),
                        k == 0, dst, ld_dst, grad, st);
      };
      TRY(run_ring(comm, ops, x, st));
    }
    TRY(pass_end(R, pass, out, diag, row_lse, col_lse, grad, st));
    if (pass == 0 && dI_ready) INFCL_CUDA_TRY(cudaEventRecord(dI_ready, st));  // dI final: callers may copy it out
  }
  if (world > 1) TRY(comm_async_check(comm));
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}

extern "C" infcl_status infcl_backward(infcl_comm comm, const void* I_local, const void* T_local, infcl_dtype dt,
                                       int64_t b, int d, float s, int rank, int world, const float* row_lse,
                                       const float* col_lse, const float* diag, const float* grad, float* dI,
                                       float* dT, void* ws, size_t ws_bytes, void* stream) {
  return backward_impl(comm, I_local, T_local, dt, b, d, s, rank, world, row_lse, col_lse, diag, grad, dI, dT, ws,
                       ws_bytes, stream, nullptr);
}

// ------------------------------------------------------------------------------------------ NT-Xent (SimCLR)
// The second workload through the same kernels (oracle/ntxent.py readings N1-N4).  With views
// Z = [A; B] the 2b x 2b similarity splits into four b x b blocks: (A, B) and its transpose hold the positives on
// their diagonal -- exactly the CLIP pair (I, T) = (A, B) -- and (A, A), (B, B) hold the self-similarities on
// theirs, excluded by self-masked launches.  Row LSEs: r_A over the rows of (A, B) and (A, A); r_B over the
// columns of (A, B) and the rows of (B, B) (the (B, B) row state seeds the column state the (A, B) pass
// accumulates into).  Loss: the CLIP expression with (r, c) = (r_A, r_B) and the same b.  Gradients: dA = the CLIP
// dI with (r, c) = (r_A, r_B) plus the self-masked pass (rows A, streamed A, LSE r_A on both sides); dB likewise.
// At world > 1 every block is a ring over the ranks with the same schedule (fwd_ring_ops / bwd_ring_ops).
namespace {
// self-similarity forward block: rows vs held views of the same side, the own block self-masked; row partials
// merged into `rstate` (the column statistics are those of the rows, by symmetry, and are not used)
infcl_status fwd_self_step(Rank& R, const __nv_bfloat16* rows, const __nv_bfloat16* held, bool own, float2* rstate,
                           cudaStream_t st) {
  PassArgs a{};
  a.A = rows;
  a.B = held;
  a.nrows = a.ncols = R.L.bs;
  a.dk = a.ld = R.L.dk;
  a.scale = R.s;
  a.self_mask = own ? 1 : 0;
  a.col_slots = R.slots();
  a.slot_ld = R.L.slot_ld;
  a.row_parts = R.rparts();
  TRY(launch_pair_forward(a, st));
  launch_merge_rows(R.rparts(), rstate, R.L.bs, fwd_geom(R.L.bs, R.L.bs), st);
  return INFCL_OK;
}

infcl_status ntxent_check(infcl_dtype dt, int world, infcl_comm comm) {
  if (dt != INFCL_BF16) return fail(INFCL_ERR_UNSUPPORTED, "NT-Xent takes bf16 views");
  if (world > 1 && !comm) return fail(INFCL_ERR_CONFIG, "world > 1 needs a communicator");
  return INFCL_OK;
}

// one self-similarity ring (world > 1): rows stationary, the same side's block travelling
infcl_status fwd_self_ring(infcl_comm comm, Rank& R, int rank, int world, const __nv_bfloat16* rows,
                           float2* rstate, cudaStream_t st) {
  std::vector<ROp> ops;
  fwd_ring_ops(world, rank, ops);
  launch_init_state(R.xstate(0), R.L.bs, st);
  RingCtx x;
  x.own = rows;
  x.owncs = R.xstate(0);
  x.bytes[XK_BLK] = (size_t)R.L.bs * R.L.dk * 2;
  x.bytes[XK_CS] = (size_t)R.L.bs * sizeof(float2);
  x.compute = [&](int k, const void* blk, const void*) {
    return fwd_self_step(R, rows, static_cast<const __nv_bfloat16*>(blk), k == 0, rstate, st);
  };
  x.merge = [](float2*) {};
  x.finish = [](const float2*) {};
  return run_ring(comm, ops, x, st);
}
}  // namespace

extern "C" infcl_status infcl_ntxent_forward(infcl_comm comm, const void* A_local, const void* B_local, infcl_dtype dt,
                                             int64_t b, int d, float s, int rank, int world, float* lse_a,
                                             float* lse_b, float* pos, float* loss, void* ws, size_t ws_bytes,
                                             void* stream) {
  const size_t need = infcl_comm_workspace_bytes(world > 1 ? comm : nullptr, b, d, world, dt);
  TRY(validate(A_local, B_local, dt, b, d, s, rank, world, ws, ws_bytes, need));
  TRY(ntxent_check(dt, world, comm));
  if (!lse_a || !lse_b || !pos || !loss) return fail(INFCL_ERR_INVALID_ARG, "null output pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PairCarveOut carve(ring_carveout(comm, world));
  Rank R;
  TRY(prepare_rank(R, A_local, B_local, dt, b, d, s, world, ws, st, world == 1 || ring_in_ws(comm)));
  if (world > 1) TRY(ring_setup(comm, R, rank, world));
  INFCL_CUDA_TRY(cudaMemsetAsync(R.acc(), 0, sizeof(double), st));
  TRY(fwd_begin(R, st));  // rstate: A views' rows; cstate(0): B views' rows
  if (world == 1) {
    TRY(fwd_self_step(R, R.B, R.B, true, R.cstate(0), st));  // (B, B)
    TRY(fwd_self_step(R, R.A, R.A, true, R.rstate(), st));   // (A, A)
    TRY(fwd_step_main(R, R.B, true, pos, st));                // (A, B): positives
    fwd_step_merge(R, R.cstate(0), st);
    fwd_finish(R, R.cstate(0), lse_a, lse_b, pos, R.acc(), st);
    launch_loss_write(R.acc(), loss, b, st);
    INFCL_CUDA_TRY(cudaGetLastError());
    return INFCL_OK;
  }
  // the (B, B) ring seeds the B rows' state, which then travels as the (A, B) ring's own column state
  TRY(fwd_self_ring(comm, R, rank, world, R.B, R.cstate(0), st));
  TRY(fwd_self_ring(comm, R, rank, world, R.A, R.rstate(), st));
  std::vector<ROp> ops;
  fwd_ring_ops(world, rank, ops);
  RingCtx x;
  x.own = R.B;
  x.owncs = R.cstate(0);
  x.bytes[XK_BLK] = (size_t)R.L.bs * R.L.dk * 2;
  x.bytes[XK_CS] = (size_t)R.L.bs * sizeof(float2);
  x.acc = R.acc();
  x.compute = [&](int k, const void* blk, const void*) {
    return fwd_step_main(R, static_cast<const __nv_bfloat16*>(blk), k == 0, pos, st);
  };
  x.merge = [&](float2* cs) { fwd_step_merge(R, cs, st); };
  x.finish = [&](const float2* cs) { fwd_finish(R, cs, lse_a, lse_b, pos, R.acc(), st); };
  TRY(run_ring(comm, ops, x, st));
  launch_loss_write(R.acc(), loss, b, st);
  TRY(comm_async_check(comm));
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}

extern "C" infcl_status infcl_ntxent_backward(infcl_comm comm, const void* A_local, const void* B_local,
                                              infcl_dtype dt, int64_t b, int d, float s, int rank, int world,
                                              const float* lse_a, const float* lse_b, const float* pos,
                                              const float* grad, float* dA, float* dB, void* ws, size_t ws_bytes,
                                              void* stream) {
  const size_t need = infcl_comm_workspace_bytes(world > 1 ? comm : nullptr, b, d, world, dt);
  TRY(validate(A_local, B_local, dt, b, d, s, rank, world, ws, ws_bytes, need));
  TRY(ntxent_check(dt, world, comm));
  if (!lse_a || !lse_b || !pos || !grad || !dA || !dB) return fail(INFCL_ERR_INVALID_ARG, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PairCarveOut carve(ring_carveout(comm, world));
  Rank R;
  TRY(prepare_rank(R, A_local, B_local, dt, b, d, s, world, ws, st, world == 1 || ring_in_ws(comm)));
  if (world > 1) TRY(ring_setup(comm, R, rank, world));
  // own2(0) = r_A, own2(1) = r_B (log2); dA starts as the exact positive-pair term of the (A, B) block
  TRY(bwd_begin(R, lse_a, lse_b, pos, grad, dA, st));
  const size_t blk_bytes = (size_t)R.L.bs * R.L.dk * 2, lse_bytes = (size_t)R.L.bs * sizeof(float);
  auto block = [&](const __nv_bfloat16* rows, const float* rows2, const __nv_bfloat16* own_blk,
                   const float* own_cols2, bool self, float* out) -> infcl_status {
    if (world == 1) return bwd_step(R, rows, rows2, own_blk, own_cols2, true, out, R.L.d, grad, st, self);
    std::vector<ROp> ops;
    bwd_ring_ops(world, rank, ops);
    RingCtx x;
    x.own = own_blk;
    x.ownl = own_cols2;
    x.bytes[XK_BLK] = blk_bytes;
    x.bytes[XK_LSE] = lse_bytes;
    x.compute = [&](int k, const void* blk, const void* lse) {
      return bwd_step(R, rows, rows2, static_cast<const __nv_bfloat16*>(blk), static_cast<const float*>(lse), k == 0,
                      out, R.L.d, grad, st, self);
    };
    return run_ring(comm, ops, x, st);
  };
  // world 1, bf16: the (A, B) block's two passes as one fused single-pass launch (dA rows and dB columns)
  bool pair_done = false;
  if (world == 1 && (R.L.gc.ok || R.L.gc3.ok)) {
    diag_init(R, 1, dB, pos, lse_a, lse_b, grad, st);
    const infcl_status fs = bwd_fused(R, dA, dB, grad, st);
    if (fs != INFCL_OK && fs != INFCL_ERR_UNSUPPORTED) return fs;
    pair_done = fs == INFCL_OK;
  }
  for (int pass = 0; pass < 2; ++pass) {
    const __nv_bfloat16* rows = pass == 0 ? R.A : R.B;
    const __nv_bfloat16* other = pass == 0 ? R.B : R.A;
    const float* rows2 = R.own2(pass);
    const float* other2 = R.own2(1 - pass);
    float* out = pass == 0 ? dA : dB;
    if (!pair_done) {
      if (pass == 1) diag_init(R, 1, dB, pos, lse_a, lse_b, grad, st);
      TRY(block(rows, rows2, other, other2, false, out));  // the other views: positives on the diagonal
    }
    TRY(block(rows, rows2, rows, rows2, true, out));  // the same side's views: self-similarity excluded
  }
  if (world > 1) TRY(comm_async_check(comm));
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}

// ------------------------------------------------------------------------------------------ virtual ring
// `world` logical ranks on one device, lock-step, blocks exchanged by device copies on the same stream.
extern "C" infcl_status infcl_forward_virtual(const void* I, const void* T, infcl_dtype dt, int64_t b, int d, float s,
                                              int world, float* row_lse, float* col_lse, float* diag, float* loss,
                                              void* ws, size_t ws_bytes, void* stream) {
  const size_t per = infcl_workspace_bytes(b, d, world, dt);
  TRY(validate(I, T, dt, b, d, s, 0, world, ws, ws_bytes, per * (size_t)world));
  if (!row_lse || !col_lse || !diag || !loss) return fail(INFCL_ERR_INVALID_ARG, "null output pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int bs = (int)(b / world);
  const size_t esz = dt == INFCL_FP32 ? 4 : 2;
  std::vector<Rank> R(world);
  for (int r = 0; r < world; ++r) {
    TRY(prepare_rank(R[r], static_cast<const uint8_t*>(I) + (size_t)r * bs * d * esz,
                     static_cast<const uint8_t*>(T) + (size_t)r * bs * d * esz, dt, b, d, s, world,
                     static_cast<uint8_t*>(ws) + (size_t)r * per, st));
    INFCL_CUDA_TRY(cudaMemsetAsync(R[r].acc(), 0, sizeof(double), st));
    TRY(fwd_begin(R[r], st));
  }
  const size_t blk_bytes = (size_t)bs * R[0].L.dk * 2, cs_bytes = (size_t)bs * sizeof(float2);
  std::vector<const __nv_bfloat16*> held(world);
  for (int r = 0; r < world; ++r) held[r] = R[r].B;
  for (int k = 0; k < world; ++k) {
    for (int r = 0; r < world; ++r) {
      TRY(fwd_step_main(R[r], held[r], k == 0, diag + (size_t)r * bs, st));
      fwd_step_merge(R[r], R[r].cstate(k & 1), st);
    }
    for (int r = 0; r < world; ++r) {  // rank r receives from r+1: block and column state
      const int src = next_rank(r, world);
      if (k + 1 < world)
        INFCL_CUDA_TRY(cudaMemcpyAsync(R[r].ring_blk(k & 1), held[src], blk_bytes, cudaMemcpyDeviceToDevice, st));
      INFCL_CUDA_TRY(cudaMemcpyAsync(R[r].cstate((k + 1) & 1) + 0, R[src].cstate(k & 1), cs_bytes,
                                     cudaMemcpyDeviceToDevice, st));
    }
    for (int r = 0; r < world; ++r) held[r] = R[r].ring_blk(k & 1);
  }
  // every logical rank adds its partial into rank 0's accumulator (the virtual all-reduce)
  for (int r = 0; r < world; ++r)
    fwd_finish(R[r], R[r].cstate(world & 1), row_lse + (size_t)r * bs, col_lse + (size_t)r * bs,
               diag + (size_t)r * bs, R[0].acc(), st);
  launch_loss_write(R[0].acc(), loss, b, st);
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}

extern "C" infcl_status infcl_backward_virtual(const void* I, const void* T, infcl_dtype dt, int64_t b, int d, float s,
                                               int world, const float* row_lse, const float* col_lse,
                                               const float* diag, const float* grad, float* dI, float* dT, void* ws,
                                               size_t ws_bytes, void* stream) {
  const size_t per = infcl_workspace_bytes(b, d, world, dt);
  TRY(validate(I, T, dt, b, d, s, 0, world, ws, ws_bytes, per * (size_t)world));
  if (!row_lse || !col_lse || !diag || !grad || !dI || !dT) return fail(INFCL_ERR_INVALID_ARG, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int bs = (int)(b / world);
  const size_t esz = dt == INFCL_FP32 ? 4 : 2;
  std::vector<Rank> R(world);
  for (int r = 0; r < world; ++r) {
    TRY(prepare_rank(R[r], static_cast<const uint8_t*>(I) + (size_t)r * bs * d * esz,
                     static_cast<const uint8_t*>(T) + (size_t)r * bs * d * esz, dt, b, d, s, world,
                     static_cast<uint8_t*>(ws) + (size_t)r * per, st));
    TRY(bwd_begin(R[r], row_lse + (size_t)r * bs, col_lse + (size_t)r * bs, diag + (size_t)r * bs, grad,
                  dI + (size_t)r * bs * d, st));
  }
  const size_t blk_bytes = (size_t)bs * R[0].L.dk * 2, lse_bytes = (size_t)bs * sizeof(float);
  if (R[0].L.gc.ok && fused_ring_enabled()) {
    // the fused ring's schedule (bwd_fused_ring_ops) on one device: rank r's step-k launch adds its dI rows and the
    // dT partial of block (r + k) mod n -- accumulated in place in that block's dT rows, in the same step order as
    // the travelling partial of the real ring
    std::vector<const __nv_bfloat16*> held(world);
    std::vector<const float*> held2(world);
    for (int r = 0; r < world; ++r) {
      held[r] = R[r].B;
      held2[r] = R[r].own2(1);
      diag_init(R[r], 1, dT + (size_t)r * bs * d, diag + (size_t)r * bs, row_lse + (size_t)r * bs,
                col_lse + (size_t)r * bs, grad, st);
    }
    for (int k = 0; k < world; ++k) {
      for (int r = 0; r < world; ++r) {
        const int blk = (r + k) % world;
        TRY(bwd_fused(R[r], dI + (size_t)r * bs * d, dT + (size_t)blk * bs * d, grad, st, held[r], held2[r], k == 0,
                      false));
      }
      if (k + 1 < world) {
        for (int r = 0; r < world; ++r) {
          const int src = next_rank(r, world);
          INFCL_CUDA_TRY(cudaMemcpyAsync(R[r].ring_blk(k & 1), held[src], blk_bytes, cudaMemcpyDeviceToDevice, st));
          INFCL_CUDA_TRY(cudaMemcpyAsync(R[r].ring_lse(k & 1), held2[src], lse_bytes, cudaMemcpyDeviceToDevice, st));
        }
        for (int r = 0; r < world; ++r) {
          held[r] = R[r].ring_blk(k & 1);
          held2[r] = R[r].ring_lse(k & 1);
        }
      }
    }
    INFCL_CUDA_TRY(cudaGetLastError());
    return INFCL_OK;
  }
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<const __nv_bfloat16*> held(world);
    std::vector<const float*> held2(world);
    for (int r = 0; r < world; ++r) {
      held[r] = pass == 0 ? R[r].B : R[r].A;
      held2[r] = R[r].own2(pass == 0 ? 1 : 0);
      if (!R[r].L.f32 && pass == 1)
        diag_init(R[r], 1, dT + (size_t)r * bs * d, diag + (size_t)r * bs, row_lse + (size_t)r * bs,
                  col_lse + (size_t)r * bs, grad, st);
    }
    for (int k = 0; k < world; ++k) {
      for (int r = 0; r < world; ++r) {
        float* out = (pass == 0 ? dI : dT) + (size_t)r * bs * d;
        TRY(bwd_step(R[r], pass == 0 ? R[r].A : R[r].B, R[r].own2(pass == 0 ? 0 : 1), held[r], held2[r], k == 0,
                     pass_dst(R[r], out), R[r].L.f32 ? R[r].L.dk : d, grad, st));
      }
      if (k + 1 < world) {
        for (int r = 0; r < world; ++r) {
          const int src = next_rank(r, world);
          INFCL_CUDA_TRY(cudaMemcpyAsync(R[r].ring_blk(k & 1), held[src], blk_bytes, cudaMemcpyDeviceToDevice, st));
          INFCL_CUDA_TRY(cudaMemcpyAsync(R[r].ring_lse(k & 1), held2[src], lse_bytes, cudaMemcpyDeviceToDevice, st));
        }
        for (int r = 0; r < world; ++r) {
          held[r] = R[r].ring_blk(k & 1);
          held2[r] = R[r].ring_lse(k & 1);
        }
      }
    }
    for (int r = 0; r < world; ++r) {
      float* out = (pass == 0 ? dI : dT) + (size_t)r * bs * d;
      TRY(pass_end(R[r], pass, out, diag + (size_t)r * bs, row_lse + (size_t)r * bs, col_lse + (size_t)r * bs, grad,
                   st));
    }
  }
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}

// ------------------------------------------------------------------------------------------ e2e host entry
extern "C" size_t infcl_e2e_scratch_bytes(int64_t b, int d, infcl_dtype dt) {
  if (b < 1 || d < 1) return 0;
  const size_t esz = dt == INFCL_FP32 ? 4 : 2;
  size_t o = 0;
  o += align_up((size_t)b * d * esz) * 2;          // I, T
  o += align_up((size_t)b * sizeof(float)) * 3;    // r, c, diag
  o += align_up(64);                               // loss, grad
  o += align_up((size_t)b * d * sizeof(float)) * 2;  // dI, dT
  o += infcl_workspace_bytes(b, d, 1, dt);
  return o;
}

extern "C" infcl_status infcl_loss_grad_host(const void* I_host, const void* T_host, infcl_dtype dt, int64_t b, int d,
                                             float s, float grad_loss, float* loss_host, float* dI_host,
                                             float* dT_host, void* scratch, size_t scratch_bytes, void* stream) {
  if (!I_host || !T_host || !loss_host || !dI_host || !dT_host || !scratch)
    return fail(INFCL_ERR_INVALID_ARG, "null pointer");
  const size_t need = infcl_e2e_scratch_bytes(b, d, dt);
  if (need == 0) return fail(INFCL_ERR_SHAPE, "bad shape");
  if (scratch_bytes < need) return fail(INFCL_ERR_WORKSPACE, "scratch too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t esz = dt == INFCL_FP32 ? 4 : 2;
  uint8_t* p = static_cast<uint8_t*>(scratch);
  auto take = [&](size_t bytes) {
    uint8_t* at = p;
    p += align_up(bytes);
    return at;
  };
  void* I = take((size_t)b * d * esz);
  void* T = take((size_t)b * d * esz);
  float* r = reinterpret_cast<float*>(take((size_t)b * 4));
  float* c = reinterpret_cast<float*>(take((size_t)b * 4));
  float* dg = reinterpret_cast<float*>(take((size_t)b * 4));
  float* lg = reinterpret_cast<float*>(take(64));
  float* dI = reinterpret_cast<float*>(take((size_t)b * d * 4));
  float* dT = reinterpret_cast<float*>(take((size_t)b * d * 4));
  void* ws = p;
  const size_t wsb = infcl_workspace_bytes(b, d, 1, dt);
  TRY(validate(I_host, T_host, dt, b, d, s, 0, 1, ws, wsb, wsb));
  // side streams for host->device (cin) and device->host (cout) copies overlapping the kernels on `st`, with
  // their events: created once per device (the call synchronises before returning, so one set per device
  // suffices; a mutex serialises concurrent host threads that share a device)
  struct CopyCtx {
    cudaStream_t cin = nullptr, cout = nullptr;
    cudaEvent_t evs[24] = {};
    std::mutex mu;
  };
  static CopyCtx ctxs[64];
  int dev = 0;
  INFCL_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(INFCL_ERR_UNSUPPORTED, "device index above 63");
  CopyCtx& cx = ctxs[dev];
  std::lock_guard<std::mutex> lock(cx.mu);
  if (!cx.cin) {
    INFCL_CUDA_TRY(cudaStreamCreateWithFlags(&cx.cin, cudaStreamNonBlocking));
    INFCL_CUDA_TRY(cudaStreamCreateWithFlags(&cx.cout, cudaStreamNonBlocking));
    for (auto& e : cx.evs) INFCL_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t cin = cx.cin, cout = cx.cout;
  cudaEvent_t* evs = cx.evs;
  const size_t row_bytes = (size_t)d * esz;
  // bf16: the stationary side is processed in row chunks so that (1) the forward starts on the first chunk of
  // I while the rest is still in flight and (2) each finished chunk of dT is copied out while the next one
  // computes (dI is copied out during the whole dT pass).  fp32 inputs run unchunked (their bf16 split needs
  // the whole block).
  const int nch = (dt == INFCL_BF16 && b >= 32768) ? 4 : 1;
  // chunk boundaries (sixteenths of b, 128-row aligned): the forward's first I chunk is small (its copy is
  // exposed), the dT pass's last chunk is small (its copy-out is exposed).  tests/test_gpu_large.py samples the
  // rows on both sides of every boundary (same formulas).
  auto at16 = [&](int e) { return std::min<int64_t>(b, (b * e / 16 + 127) / 128 * 128); };
  // Forward on 4 I row chunks x 2 T column pieces as their copies land.  The available work grows with the
  // product of the arrived rows and columns, so the first pieces are small: I in sixteenths {1, 3, 6, 6} and T
  // in {3/8, 5/8}, copied T0 I0 I1 I2 T1 I3, blocks run in readiness order (timeline model at 55-128 GB/s:
  // the forward ends 0.13-0.54 ms earlier than with I in eighths {1, 3, 2, 2}, T in halves, T0 I0 T1 I1 I2 I3,
  // row-major blocks; measured -0.7 %).
  const int64_t fwd_cut[5] = {0, at16(1), at16(4), at16(10), b};
  // dT pass chunks: the last one's copy-out is exposed, so it is small (sixteenths {6, 5, 4, 1})
  const int64_t dT_cut[5] = {0, at16(6), at16(11), at16(15), b};
  const int64_t tsplit = std::min<int64_t>(b, (b * 3 / 8 + 255) / 256 * 256);
  auto cols_of = [&](int h, int64_t& c0, int64_t& c1) {
    c0 = h == 0 ? 0 : tsplit;
    c1 = h == 0 ? tsplit : b;
  };
  INFCL_CUDA_TRY(cudaEventRecord(evs[0], st));  // scratch is free once prior work on `st` is done
  INFCL_CUDA_TRY(cudaStreamWaitEvent(cin, evs[0], 0));
  INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[0], 0));
  auto copy_in = [&](void* dst, const void* src, int64_t r0, int64_t r1) -> infcl_status {
    if (r1 > r0)
      INFCL_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + r0 * row_bytes,
                                     static_cast<const uint8_t*>(src) + r0 * row_bytes, (r1 - r0) * row_bytes,
                                     cudaMemcpyHostToDevice, cin));
    return INFCL_OK;
  };
  if (nch == 1) {
    TRY(copy_in(T, T_host, 0, b));
    TRY(copy_in(I, I_host, 0, b));
    INFCL_CUDA_TRY(cudaEventRecord(evs[2], cin));
  } else {  // copy order T0, I0, I1, I2, T1, I3; events: T0 1, I_k 2+k, T1 7
    int64_t c0, c1;
    cols_of(0, c0, c1);
    TRY(copy_in(T, T_host, c0, c1));
    INFCL_CUDA_TRY(cudaEventRecord(evs[1], cin));
    for (int k = 0; k < nch; ++k) {
      TRY(copy_in(I, I_host, fwd_cut[k], fwd_cut[k + 1]));
      INFCL_CUDA_TRY(cudaEventRecord(evs[2 + k], cin));
      if (k == 2) {
        cols_of(1, c0, c1);
        TRY(copy_in(T, T_host, c0, c1));
        INFCL_CUDA_TRY(cudaEventRecord(evs[7], cin));
      }
    }
  }
  launch_set_scalar(lg + 1, grad_loss, st);
  if (nch == 1) {
    INFCL_CUDA_TRY(cudaStreamWaitEvent(st, evs[2], 0));
    TRY(infcl_forward(nullptr, I, T, dt, b, d, s, 0, 1, r, c, dg, lg, ws, wsb, stream));
    INFCL_CUDA_TRY(cudaEventRecord(evs[8], st));
    INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[8], 0));
    INFCL_CUDA_TRY(cudaMemcpyAsync(loss_host, lg, sizeof(float), cudaMemcpyDeviceToHost, cout));
    TRY(backward_impl(nullptr, I, T, dt, b, d, s, 0, 1, r, c, dg, lg + 1, dI, dT, ws, wsb, stream, evs[9]));
    INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[9], 0));
    INFCL_CUDA_TRY(cudaMemcpyAsync(dI_host, dI, (size_t)b * d * 4, cudaMemcpyDeviceToHost, cout));
    INFCL_CUDA_TRY(cudaEventRecord(evs[10], st));
    INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[10], 0));
    INFCL_CUDA_TRY(cudaMemcpyAsync(dT_host, dT, (size_t)b * d * 4, cudaMemcpyDeviceToHost, cout));
  } else {
    Rank R;
    TRY(prepare_rank(R, I, T, dt, b, d, s, 1, ws, st));
    INFCL_CUDA_TRY(cudaMemsetAsync(R.acc(), 0, sizeof(double), st));
    TRY(fwd_begin(R, st));
    fwd_blocks_begin(R, st);
    // block order (I chunk, T piece): readiness order for the copy order above
    static const int kOrder[8][2] = {{0, 0}, {1, 0}, {2, 0}, {0, 1}, {1, 1}, {2, 1}, {3, 0}, {3, 1}};
    for (int i = 0; i < 2 * nch; ++i) {
      const int k = kOrder[i][0], h = kOrder[i][1];
      const int64_t r0 = fwd_cut[k], r1 = fwd_cut[k + 1];
      int64_t c0, c1;
      cols_of(h, c0, c1);
      INFCL_CUDA_TRY(cudaStreamWaitEvent(st, evs[2 + k], 0));           // rows [r0, r1) of I
      INFCL_CUDA_TRY(cudaStreamWaitEvent(st, evs[h == 0 ? 1 : 7], 0));  // columns [c0, c1) of T
      if (r1 > r0 && c1 > c0) TRY(fwd_block(R, (int)r0, (int)r1, (int)c0, (int)c1, dg, st));
    }
    fwd_blocks_finish(R, st);
    fwd_finish(R, R.cstate(0), r, c, dg, R.acc(), st);
    launch_loss_write(R.acc(), lg, b, st);
    INFCL_CUDA_TRY(cudaEventRecord(evs[8], st));
    INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[8], 0));
    INFCL_CUDA_TRY(cudaMemcpyAsync(loss_host, lg, sizeof(float), cudaMemcpyDeviceToHost, cout));
    // Hybrid backward (INFCL_E2E_HYBRID, default on): one fused single-pass launch over I rows [0, f) x all T
    // columns (dI rows [0, f) final, their dT contributions accumulated), then the two-pass pieces restricted to
    // the remaining I rows [f, b): the dI pass over them, and the dT pass in T-row chunks streaming only those I
    // rows -- gradient rows still finish progressively for the copy-out, and the first half of the work runs at the
    // fused kernel's rate.  Otherwise: the dI pass (whole), then dI copied out while the dT pass runs chunk by chunk.
    static const bool hybrid = [] {
      const char* e = getenv("INFCL_E2E_HYBRID");
      return !(e && atoi(e) == 0);
    }();
    // the fused part: 8/16 of b (A/B over 5-12 sixteenths, scripts/experiments/e2e_fsplit.sh: 8 best; the tests
    // sample the rows around this split, tests/test_gpu_large.py e2e_boundaries); INFCL_E2E_FSPLIT overrides
    static const int fsix = [] {
      const char* e = getenv("INFCL_E2E_FSPLIT");
      return e ? std::max(1, std::min(15, atoi(e))) : 8;
    }();
    const int64_t fsplit = at16(fsix);
    if (hybrid && fsplit < b && gc_plan((int)fsplit, R.L.bs, R.L.dk).ok) {
      TRY(bwd_begin(R, r, c, dg, lg + 1, dI, st));
      diag_init(R, 1, dT, dg, r, c, lg + 1, st);
      const float coef = (float)((double)R.s / (2.0 * (double)R.b));
      PassArgs fa{};
      fa.A = R.A;
      fa.B = R.B;
      fa.nrows = (int)fsplit;
      fa.ncols = R.L.bs;
      fa.dk = fa.ld = R.L.dk;
      fa.scale = R.s;
      fa.diag_on = 1;
      fa.lse_row2 = R.own2(0);
      fa.lse_col2 = R.own2(1);
      fa.dA = dI;
      fa.ld_dA = R.L.d;
      fa.d_out = R.L.dk;
      fa.grad = lg + 1;
      fa.coef_base = coef;
      fa.dB = dT;
      fa.ld_dB = R.L.d;
      fa.gc_ws = R.ws + R.L.off_slots;
      fa.gc_ws_bytes = R.L.gc_bytes();
      const infcl_status fs = launch_pair_backward_fused(fa, st);
      if (fs == INFCL_OK) {
        INFCL_CUDA_TRY(cudaEventRecord(evs[9], st));
        INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[9], 0));
        INFCL_CUDA_TRY(cudaMemcpyAsync(dI_host, dI, (size_t)fsplit * d * 4, cudaMemcpyDeviceToHost, cout));
        // dI pass over I rows [f, b): stationary rows f.., all T columns; the positive pair of local row i is column
        // f + i
        PassArgs da{};
        da.A = R.A + (size_t)fsplit * R.L.dk;
        da.B = R.B;
        da.nrows = (int)(b - fsplit);
        da.ncols = R.L.bs;
        da.dk = da.ld = R.L.dk;
        da.scale = R.s;
        da.diag_on = 1;
        da.row_off = (int)fsplit;
        da.lse_row2 = R.own2(0) + fsplit;
        da.lse_col2 = R.own2(1);
        da.dA = dI + (size_t)fsplit * d;
        da.ld_dA = R.L.d;
        da.d_out = R.L.dk;
        da.grad = lg + 1;
        da.coef_base = coef;
        da.tail_scratch = R.tails();
        TRY(launch_pair_backward(da, st));
        INFCL_CUDA_TRY(cudaEventRecord(evs[10], st));
        INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[10], 0));
        INFCL_CUDA_TRY(cudaMemcpyAsync(dI_host + (size_t)fsplit * d, dI + (size_t)fsplit * d,
                                       (size_t)(b - fsplit) * d * 4, cudaMemcpyDeviceToHost, cout));
        // dT pass in T-row chunks over the remaining I rows [f, b) (the fused launch added rows [0, f)); the positive
        // pair of T row j is streamed column j - f
        for (int k = 0; k < nch; ++k) {
          const int r0 = (int)dT_cut[k], r1 = (int)dT_cut[k + 1];
          if (r1 <= r0) continue;
          PassArgs ta{};
          ta.A = R.B + (size_t)r0 * R.L.dk;
          ta.B = R.A + (size_t)fsplit * R.L.dk;
          ta.nrows = r1 - r0;
          ta.ncols = (int)(b - fsplit);
          ta.dk = ta.ld = R.L.dk;
          ta.scale = R.s;
          ta.diag_on = 1;
          ta.row_off = r0 - (int)fsplit;
          ta.lse_row2 = R.own2(1) + r0;
          ta.lse_col2 = R.own2(0) + fsplit;
          ta.dA = dT + (size_t)r0 * d;
          ta.ld_dA = R.L.d;
          ta.d_out = R.L.dk;
          ta.grad = lg + 1;
          ta.coef_base = coef;
          ta.tail_scratch = R.tails();
          TRY(launch_pair_backward(ta, st));
          INFCL_CUDA_TRY(cudaEventRecord(evs[12 + k], st));
          INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[12 + k], 0));
          INFCL_CUDA_TRY(cudaMemcpyAsync(dT_host + (size_t)r0 * d, dT + (size_t)r0 * d, (size_t)(r1 - r0) * d * 4,
                                         cudaMemcpyDeviceToHost, cout));
        }
        INFCL_CUDA_TRY(cudaEventRecord(evs[20], cout));
        INFCL_CUDA_TRY(cudaStreamWaitEvent(st, evs[20], 0));  // the call's stream orders after every copy
        INFCL_CUDA_TRY(cudaStreamSynchronize(st));
        return INFCL_OK;
      }
      if (fs != INFCL_ERR_UNSUPPORTED) return fs;
      // not all CTA pairs co-resident: the two passes below (they re-initialise dI and dT)
    }
    TRY(bwd_begin(R, r, c, dg, lg + 1, dI, st));
    TRY(bwd_step(R, R.A, R.own2(0), R.B, R.own2(1), true, dI, d, lg + 1, st));
    TRY(pass_end(R, 0, dI, dg, r, c, lg + 1, st));
    INFCL_CUDA_TRY(cudaEventRecord(evs[9], st));
    INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[9], 0));
    INFCL_CUDA_TRY(cudaMemcpyAsync(dI_host, dI, (size_t)b * d * 4, cudaMemcpyDeviceToHost, cout));
    diag_init(R, 1, dT, dg, r, c, lg + 1, st);
    for (int k = 0; k < nch; ++k) {
      const int r0 = (int)dT_cut[k], r1 = (int)dT_cut[k + 1];
      if (r1 <= r0) continue;
      TRY(bwd_dT_chunk(R, r0, r1, lg + 1, dT, st));
      INFCL_CUDA_TRY(cudaEventRecord(evs[12 + k], st));
      INFCL_CUDA_TRY(cudaStreamWaitEvent(cout, evs[12 + k], 0));
      INFCL_CUDA_TRY(cudaMemcpyAsync(dT_host + (size_t)r0 * d, dT + (size_t)r0 * d, (size_t)(r1 - r0) * d * 4,
                                     cudaMemcpyDeviceToHost, cout));
    }
  }
  INFCL_CUDA_TRY(cudaEventRecord(evs[20], cout));
  INFCL_CUDA_TRY(cudaStreamWaitEvent(st, evs[20], 0));  // the call's stream orders after every copy
  INFCL_CUDA_TRY(cudaStreamSynchronize(st));
  return INFCL_OK;
}

extern "C" uint64_t infcl_launch_count(void) { return launch_counter(); }
extern "C" void infcl_reset_launch_count(void) { launch_counter() = 0; }

extern "C" void infcl_profile_enable(int on) { profile_enable(on != 0); }
extern "C" infcl_status infcl_profile_read(int kind, int* launches, double* total_ms) {
  return profile_read(kind, launches, total_ms);
}

extern "C" infcl_status infcl_grad_scale_partial(const void* I_local, const float* dI_local, infcl_dtype dt,
                                                 int64_t rows, int d, float s, double* out, void* stream) {
  if (!I_local || !dI_local || !out) return fail(INFCL_ERR_INVALID_ARG, "null pointer");
  if (dt != INFCL_BF16 && dt != INFCL_FP32) return fail(INFCL_ERR_INVALID_ARG, "bad dtype");
  if (!(s > 0.f) || !std::isfinite(s)) return fail(INFCL_ERR_INVALID_ARG, "logit scale must be finite and > 0");
  if (rows < 1 || d < 1) return fail(INFCL_ERR_SHAPE, "rows and d must be >= 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  INFCL_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st));
  launch_grad_scale(I_local, dt == INFCL_FP32, dI_local, (long long)rows * d, 1.0 / (double)s, out, st);
  INFCL_CUDA_TRY(cudaGetLastError());
  return INFCL_OK;
}
