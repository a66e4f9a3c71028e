/*
 * infcl.h -- C ABI of the B200-native Inf-CL loss hot path (arXiv 2410.17243).
 *
 * The library computes the symmetric image-text InfoNCE loss and its gradients tile by tile, never
 * materialising the b x b similarity matrix, on sm_100a (B200) tensor cores, and runs it as a ring over the
 * GPUs of one box.  Citations: "P:n" = PAPER.md line n (section / equation / algorithm in brackets).
 *
 *   x_ij = s * <I_i, T_j>                                   [P:91, Eq.1; temperature omitted by the paper]
 *   r_i  = log sum_j exp(x_ij)     (image->text LSE, the paper's l)       [Eq.2, Eq.3-5 P:119-160]
 *   c_j  = log sum_i exp(x_ij)     (text->image LSE)                      ["symmetric", P:85]
 *   L    = ( mean_i (r_i - x_ii) + mean_j (c_j - x_jj) ) / 2              [Eq.2, reading Q4]
 *   G_ij = g/(2b) (e^{x_ij - r_i} + e^{x_ij - c_j}) - (g/b) [i==j]        [Eq.6-8 P:166-188]
 *   dI   = s G T,   dT = s G^T I                                          [Eq.7, Alg.3/4 P:539-599]
 *
 * Layout and ownership (all calls): every pointer argument is caller-owned DEVICE memory (for the
 * *_host entry points: HOST memory) that must stay valid until the stream work completes; the library
 * never allocates device memory on the hot path (the caller passes a workspace of
 * infcl_workspace_bytes()).  Feature shards are row-major [b/world][d], d contiguous, 16-byte aligned
 * rows (d % 8 == 0), dtype bf16 (INFCL_BF16) or fp32 (INFCL_FP32).  LSE/diag vectors are fp32 [b/world],
 * natural log.  Gradients are fp32 [b/world][d].  Rank r owns global rows [r*b/world, (r+1)*b/world) of
 * both I and T (Alg.1); the positive pair of row i is column i (reading Q18).
 *
 * Errors: arguments are validated synchronously before any launch and a status is returned; the detail
 * string is available from infcl_last_error() (thread-local).  Execution is asynchronous and ordered on
 * `stream` (a cudaStream_t passed as void*).  Calls with world > 1 are collective over the ring of `comm`:
 * every rank must call with identical (b, d, s, world) or the ring deadlocks, as NCCL would.
 * NaN inputs propagate to NaN outputs.  There is no CPU fallback and no second backend: on a device other
 * than sm_100 the calls fail with INFCL_ERR_UNSUPPORTED.
 */
#ifndef INFCL_H_
#define INFCL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  INFCL_OK = 0,
  INFCL_ERR_INVALID_ARG = 1, /* null pointer, non-finite or negative scale, bad dtype            */
  INFCL_ERR_SHAPE = 2,       /* b < 1, d < 1, d % 8 != 0, d above the kernel limit (768; 256 fp32) */
  INFCL_ERR_CONFIG = 3,      /* b % world != 0, rank out of range, comm mismatch     */
  INFCL_ERR_CUDA = 4,        /* a CUDA runtime/driver call failed                                 */
  INFCL_ERR_NCCL = 5,        /* an NCCL call failed or libnccl could not be loaded                */
  INFCL_ERR_WORKSPACE = 6,   /* workspace null / smaller than infcl_workspace_bytes()             */
  INFCL_ERR_UNSUPPORTED = 7  /* device is not sm_100 (B200)                                       */
} infcl_status;

typedef enum { INFCL_BF16 = 0, INFCL_FP32 = 1 } infcl_dtype;

/* Opaque ring communicator: a transport, a communication stream and events.  NULL for world==1. */
typedef struct infcl_comm_s* infcl_comm;

/* Ring transports.  NCCL: grouped ncclSend/ncclRecv (the receive buffers are in the caller's workspace).
 * IPC: one-sided copy-engine writes into the peer's library-owned receive region over CUDA IPC mappings
 * (NVLink/NVSwitch peer memory across GPUs; also valid when several ranks share one GPU), synchronised by
 * stream memory operations on 32-bit fill/release counters.  Across GPUs the peer copies run on the copy
 * engines, so the exchange can overlap the persistent compute kernels that occupy every SM (an NCCL kernel
 * must wait for an SM); same-device copies do not overlap them (measured). */
typedef enum { INFCL_TRANSPORT_NCCL = 0, INFCL_TRANSPORT_IPC = 1 } infcl_transport;

const char* infcl_status_string(infcl_status s);
/* Thread-local detail of the last failing call on this thread (e.g. "b=7 not divisible by world=2"). */
const char* infcl_last_error(void);
/* Library version: major*10000 + minor*100 + patch. */
int infcl_version(void);

/* ---------------------------------------------------------------------------------------------------
 * Ring communicator (Alg.1 / Alg.3 cross-GPU tiling).
 * infcl_get_unique_id: rank 0 writes a 128-byte NCCL unique id to host memory `id128`; the caller
 *   broadcasts it (torch.distributed) to all ranks.
 * infcl_comm_init: collective; `device` is the CUDA ordinal of this rank.  libnccl.so.2 is loaded lazily.
 * ------------------------------------------------------------------------------------------------- */
infcl_status infcl_get_unique_id(void* id128);
infcl_status infcl_comm_init(infcl_comm* out, int rank, int world, const void* id128, int device);
infcl_status infcl_comm_destroy(infcl_comm comm);

/* IPC transport (the same ring schedule, Q13/Q14/Q15 readings; P:216-219 overlap):
 * infcl_comm_init_ipc: allocates and zeroes this rank's receive region on `device` (2 slots each of one
 *   travelling block [max_b/world][d'] bf16 (d' = 3 max_d for fp32 inputs), one column state, one LSE vector and,
 *   for bf16, one travelling dT partial [max_b/world][max_d] fp32 (the fused backward ring), plus a 4-KB counter
 *   page; infcl_comm_ipc_region_bytes reports its size).  The region is the one device
 *   allocation the library owns; it is freed by infcl_comm_destroy.  2 <= world <= 64.
 * infcl_comm_ipc_handle: writes the region's 64-byte cudaIpcMemHandle_t to host memory `handle64`.
 * infcl_comm_ipc_connect: `handles` = world x 64 bytes (host), rank q's handle at offset 64 q, as gathered
 *   by the caller (torch.distributed all_gather); maps every peer region.  Must precede the first call.
 * Errors: INFCL_ERR_UNSUPPORTED without stream memory operations; INFCL_ERR_CUDA on IPC failures;
 *   INFCL_ERR_WORKSPACE when a call's shard exceeds the region's (max_b, max_d). */
infcl_status infcl_comm_init_ipc(infcl_comm* out, int rank, int world, int device, int64_t max_b, int max_d,
                                 infcl_dtype dt);
infcl_status infcl_comm_ipc_handle(infcl_comm comm, void* handle64);
infcl_status infcl_comm_ipc_connect(infcl_comm comm, const void* handles);
/* Collective self-test of a connected IPC comm: each rank copies 256 B into rank r-1's region and bumps its
 * counter (the ring's copy, remote-write and wait paths), then verifies the bytes it received from r+1.
 * Returns INFCL_ERR_CUDA (instead of hanging a later call) when a peer path fails or does not complete within
 * timeout_ms.  Call once per communicator, after infcl_comm_ipc_connect on every rank. */
infcl_status infcl_comm_ipc_selftest(infcl_comm comm, int timeout_ms);
size_t infcl_comm_ipc_region_bytes(infcl_comm comm);
/* INFCL_TRANSPORT_NCCL / INFCL_TRANSPORT_IPC, or -1 for NULL */
int infcl_comm_transport(infcl_comm comm);

/* The per-rank ring schedule (host only, no device): the op list infcl_forward (which = 0), one two-pass
 * infcl_backward pass (which = 1) or the fused single-pass backward whose dT partials travel (which = 2) executes
 * at world > 1, as int32 records of 6 {code, a, b, c, tag, 0} (codes,
 * streams and buffer references in api.cu: OP_*, RS_*, BUF_*; slot reference = 2 * kind + s).  Writes at most
 * `cap` records to `out` (may be NULL) and returns the count, or -1 for bad arguments.  tests/test_ring_schedule.py
 * replays it for n ranks under both transports' semantics to check it is race- and deadlock-free. */
int infcl_ring_schedule(int world, int rank, int which, int32_t* out, int cap);

/* Bytes of device workspace infcl_forward/infcl_backward need for this configuration (0 on bad args), for the
 * NCCL transport (or world == 1).  infcl_comm_workspace_bytes: the same for the transport of `comm` (the IPC
 * transport receives into its own region, so its workspace holds no ring buffers); comm may be NULL. */
size_t infcl_workspace_bytes(int64_t b, int d, int world, infcl_dtype dt);
size_t infcl_comm_workspace_bytes(infcl_comm comm, int64_t b, int d, int world, infcl_dtype dt);

/* ---------------------------------------------------------------------------------------------------
 * infcl_forward -- Alg.1 over Alg.2, plus the symmetric column direction.
 *   I_local, T_local : [b/world][d] features of this rank (device, dtype dt)
 *   b                : GLOBAL batch size; d: feature dim; logit_scale: s (fp32, finite, >= 0)
 *   row_lse, col_lse : out [b/world] fp32: r_i for this rank's image rows, c_j for its text rows
 *   diag             : out [b/world] fp32: x_ii for this rank's rows (saved for the backward)
 *   loss             : out device fp32 scalar: the GLOBAL symmetric mean loss L (same on every rank)
 *   workspace        : device scratch of >= infcl_workspace_bytes(b, d, world, dt) bytes, 256-B aligned
 *   comm             : ring communicator for world > 1 (NULL for world == 1)
 * ------------------------------------------------------------------------------------------------- */
infcl_status infcl_forward(infcl_comm comm, const void* I_local, const void* T_local, infcl_dtype dt, int64_t b,
                           int d, float logit_scale, int rank, int world, float* row_lse, float* col_lse,
                           float* diag, float* loss, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------------
 * infcl_backward -- Alg.3 over Alg.4: recompute each tile from the saved LSEs.  bf16 inputs: ONE fused
 *   single pass per ring step (S, G and dI on producer SMs; dT from a global ring of G tiles on consumer SMs);
 *   at world > 1 each block's dT partial travels with the block (Alg.3's rotating partials) and is home after n
 *   hops.  fp32 inputs (and INFCL_FUSED_BWD=0 / INFCL_FUSED_RING=0): two passes, dI then dT, nothing but the
 *   bf16 blocks and LSEs travels.
 *   row_lse, col_lse, diag : the forward's outputs for this rank (device fp32 [b/world])
 *   grad_loss              : device fp32 scalar g = dOut/dL (the same on every rank)
 *   dI_local, dT_local     : out [b/world][d] fp32 = g * dL/dI, g * dL/dT for this rank's rows (overwritten)
 * ------------------------------------------------------------------------------------------------- */
infcl_status infcl_backward(infcl_comm comm, const void* I_local, const void* T_local, infcl_dtype dt, int64_t b,
                            int d, float logit_scale, int rank, int world, const float* row_lse,
                            const float* col_lse, const float* diag, const float* grad_loss, float* dI_local,
                            float* dT_local, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------------
 * infcl_ntxent_forward / infcl_ntxent_backward -- the single-modality NT-Xent loss (SimCLR; self-supervised
 * learning is the paper's second named application), on the same kernels.
 * Views: A_local, B_local [b/world][d] bf16 (the two augmented views of this rank's examples; rank r owns
 * examples [r*b/world, (r+1)*b/world)); b = GLOBAL number of examples (2b views).  With Z = [A; B] and
 * x_kk' = s <z_k, z_k'>, every view's positive is the other view of its example and its own similarity is
 * excluded (oracle/ntxent.py readings N1-N3):
 *   lse_a[i], lse_b[i] = LSE over the 2b - 1 other views of A_i, B_i   (out, fp32 [b/world])
 *   pos[i]             = x(A_i, B_i) = s <A_i, B_i>                       (out, fp32 [b/world])
 *   loss               = (1/2b) sum over all 2b views of (lse - pos)       (out, device fp32 scalar, every rank)
 *   dA, dB             = g dL/dA, g dL/dB for this rank's examples        (out, fp32 [b/world][d], overwritten)
 * The 2b x 2b similarity runs as four b x b blocks: (A, B) is the CLIP pair (positives on its diagonal), (A, A)
 * and (B, B) are self-masked; at world > 1 each block is a ring over `comm` (collective, as infcl_forward).
 * Workspace: infcl_comm_workspace_bytes(comm, b, d, world, INFCL_BF16).  fp32 views: INFCL_ERR_UNSUPPORTED.
 * ------------------------------------------------------------------------------------------------- */
infcl_status infcl_ntxent_forward(infcl_comm comm, const void* A_local, const void* B_local, infcl_dtype dt, int64_t b,
                                  int d, float logit_scale, int rank, int world, float* lse_a, float* lse_b,
                                  float* pos, float* loss, void* workspace, size_t ws_bytes, void* stream);
infcl_status infcl_ntxent_backward(infcl_comm comm, const void* A_local, const void* B_local, infcl_dtype dt,
                                   int64_t b, int d, float logit_scale, int rank, int world, const float* lse_a,
                                   const float* lse_b, const float* pos, const float* grad_loss, float* dA_local,
                                   float* dB_local, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------------
 * infcl_grad_scale_partial -- g * dL/ds for a learnable logit scale (temperature, the
 * CLIP convention of P:91's omitted temperature).  x_ij = s <I_i, T_j> is bilinear, so over the global batch
 * s * dL/ds = sum_i <dI_i, I_i> exactly (pinned: tests/test_oracle_pins.py::test_scale_identity).
 *   I_local [rows][d] (dtype dt), dI_local [rows][d] fp32 (this rank's infcl_backward output, already scaled
 *   by g); out: device fp64 scalar, overwritten with sum_{i in shard} <dI_i, I_i> / s.  Callers sum the
 *   partials over ranks (one scalar all-reduce).  s must be > 0 (INFCL_ERR_INVALID_ARG otherwise).
 * ------------------------------------------------------------------------------------------------- */
infcl_status infcl_grad_scale_partial(const void* I_local, const float* dI_local, infcl_dtype dt, int64_t rows, int d,
                                      float logit_scale, double* out, void* stream);

/* ---------------------------------------------------------------------------------------------------
 * Virtual ring (test/diagnostic): runs the same per-rank ring schedule for `world` logical ranks on ONE
 * device, exchanging blocks with device copies instead of NCCL.  Arguments are the full global batch:
 * I, T [b][d]; row_lse, col_lse, diag [b]; dI, dT [b][d].  Workspace: infcl_workspace_bytes(b, d, world, dt)
 * per logical rank times `world`.
 * ------------------------------------------------------------------------------------------------- */
infcl_status infcl_forward_virtual(const void* I, const void* T, infcl_dtype dt, int64_t b, int d,
                                   float logit_scale, int world, float* row_lse, float* col_lse, float* diag,
                                   float* loss, void* workspace, size_t ws_bytes, void* stream);
infcl_status infcl_backward_virtual(const void* I, const void* T, infcl_dtype dt, int64_t b, int d,
                                    float logit_scale, int world, const float* row_lse, const float* col_lse,
                                    const float* diag, const float* grad_loss, float* dI, float* dT,
                                    void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------------
 * End-to-end convenience entry (world == 1): HOST inputs and outputs, device scratch allocated by the
 * caller.  Copies I, T host->device, runs forward + backward, copies loss, dI, dT device->host, and
 * synchronises `stream` before returning.  dev_scratch must hold infcl_e2e_scratch_bytes(b, d, dt).
 * For bf16 and b >= 32768 the copies run on library-owned side streams (one set per device, calls on the
 * same device serialise) and are pipelined against the kernels: the forward runs in blocks (I row chunks x
 * T column halves) as their inputs land, dI is copied out during the dT pass, and the dT pass runs in row
 * chunks each copied out while the next computes.  Pinned host buffers are needed for the copies to overlap
 * (pageable memory still works, synchronously).  Results equal the device entry points' up to the order
 * of the column-LSE merges (fp32 rounding).
 * ------------------------------------------------------------------------------------------------- */
size_t infcl_e2e_scratch_bytes(int64_t b, int d, infcl_dtype dt);
infcl_status infcl_loss_grad_host(const void* I_host, const void* T_host, infcl_dtype dt, int64_t b, int d,
                                  float logit_scale, float grad_loss, float* loss_host, float* dI_host,
                                  float* dT_host, void* dev_scratch, size_t scratch_bytes, void* stream);

/* Ring schedule (pure host function, no device work): block index held by `rank` at 0-based `step`,
 * k = (rank + step) mod world == Alg.3's k = (i + j - 1) mod n with 1-based j (reading Q13).
 * Returns -1 on out-of-range arguments. */
int infcl_ring_block(int rank, int world, int step);

/* Number of CUDA kernels the library launched on this thread since the last reset (for bench.py). */
uint64_t infcl_launch_count(void);
void infcl_reset_launch_count(void);

/* Kernel and ring timing for bench.py / diagnostics.  While enabled, every fused pair-kernel launch is bracketed
 * by CUDA events on its launch stream (kind 0 = forward pair kernel, kind 1 = backward pair kernel), and every
 * travelling-block hop of a ring call (world > 1) by events on the communicator's stream (kind 2: the transfer
 * as the comm stream executes it, including its wait for the receiver's slot release).
 * infcl_profile_read waits for the recorded events and returns the launch count and the summed device
 * milliseconds since the last infcl_profile_enable(1).  Single-threaded use only. */
void infcl_profile_enable(int on);
infcl_status infcl_profile_read(int kind, int* launches, double* total_ms);

#ifdef __cplusplus
}
#endif
#endif /* INFCL_H_ */
