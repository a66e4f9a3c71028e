// Thin sm_100a PTX wrappers: mbarrier, cluster, TMA, tcgen05 (UMMA / TMEM).
// Written for this library; instruction forms follow the PTX ISA as exposed by CUDA 12.9
// (cross-checked against the CUTLASS headers bundled in the image, cute/arch/*sm100*.hpp).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cstdio>

namespace infcl {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ cluster
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// map a local shared::cta address to the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on the barrier at the same smem offset in CTA `rank` of the cluster (default .release.cta semantics,
// as CUTLASS's ClusterBarrier::arrive(cta_id); data hand-offs are ordered by the caller's fences)
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t a = mapa(smem_u32(bar), rank);
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// INFCL_TRYWAIT_HINT: optional suspend-time hint (ns) of try_wait; with a hint ptxas inserts NANOSLEEP.SYNCS
// between probes, without one the probe loop spins on SYNCS.PHASECHK.TRYWAIT (A/B: scripts/build_variant.py)
#ifdef INFCL_TRYWAIT_HINT
#define INFCL_TW_SUFFIX ", " INFCL_STR(INFCL_TRYWAIT_HINT)
#else
#define INFCL_TW_SUFFIX ""
#endif
#define INFCL_STR2(x) #x
#define INFCL_STR(x) INFCL_STR2(x)
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2" INFCL_TW_SUFFIX ";\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// acquire at cluster scope so remote arrivals' prior writes are visible
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2" INFCL_TW_SUFFIX ";\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// Deadlock watchdog: a wait that has not completed after ~2^35 cycles (~17 s) reports the barrier
// (tag, block, thread, parity) and traps, so a protocol bug fails loudly instead of hanging the device.
#ifndef INFCL_WATCHDOG_CYCLES
#define INFCL_WATCHDOG_CYCLES (1ull << 35)
#endif
static __device__ __noinline__ void watchdog_fire(int tag, uint32_t parity) {
  printf("infcl watchdog: barrier tag=%d parity=%u stuck in block %d thread %d\n", tag, parity, (int)blockIdx.x,
         (int)threadIdx.x);
  __trap();
}
// non-blocking probe (test_wait never suspends the thread): the spin variants below poll it
__device__ __forceinline__ bool mbar_test_wait(uint32_t addr, uint32_t parity, bool cluster) {
  uint32_t ok;
  if (cluster)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int tag = 0) {
  uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  const unsigned long long t0 = clock64();
  while (!mbar_try_wait(a, parity)) {
    if (clock64() - t0 > INFCL_WATCHDOG_CYCLES) watchdog_fire(tag, parity);
  }
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity, int tag = 0) {
  uint32_t a = smem_u32(bar);
  if (mbar_try_wait_cluster(a, parity)) return;
  const unsigned long long t0 = clock64();
  while (!mbar_try_wait_cluster(a, parity)) {
    if (clock64() - t0 > INFCL_WATCHDOG_CYCLES) watchdog_fire(tag, parity);
  }
}

// ------------------------------------------------------------------ fences / named barriers
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 1-CTA 2D tile load, completion on a local barrier
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// CTA-pair 2D tile load: data lands in the issuing CTA's smem, transaction bytes are counted on the
// barrier at the same offset in the pair's even (leader) CTA.
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                                                 int32_t c1) {
  uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(b), "r"(c0), "r"(c1)
      : "memory");
}

// L2 cache policies for the .L2::cache_hint forms below
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_pair_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                                                      int32_t c1, uint64_t policy) {
  uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(b), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* m, const void* src, int32_t c0, int32_t c1,
                                                  uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(policy)
               : "memory");
}
// 2D tile store smem -> global (bulk async-group completion): the fused backward's G ring
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
// smem box += into global (tensor map element type, here f32), bulk async-group completion
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* m, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void st_shared_v4f(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N of this thread's most recent bulk groups still reading their smem source / not yet complete
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// drop a 128-B L2 line without writing it back (its data are dead: a consumed G ring tile)
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(p)) : "memory");
}
// bulk prefetch of [p, p + bytes) into L2 (bytes a multiple of 16)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)), "r"(bytes)
               : "memory");
}
// order generic-proxy global accesses against async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire_cta_shared(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_cta_shared_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ long long ld_volatile_shared(const long long* p) {
  long long v;
  asm volatile("ld.volatile.shared::cta.s64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_shared(long long* p, long long v) {
  asm volatile("st.volatile.shared::cta.s64 [%0], %1;" ::"r"(smem_u32(p)), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ------------------------------------------------------------------ tcgen05: TMEM allocation
template <int NCTA>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  if constexpr (NCTA == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
}
template <int NCTA>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  if constexpr (NCTA == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
  else
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ------------------------------------------------------------------ tcgen05: MMA (kind::f16, bf16 in, fp32 acc)
// D[tmem] (+)= A[smem] * B[smem]^T, described by 64-bit smem descriptors and a 32-bit instruction descriptor.
template <int NCTA>
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  if constexpr (NCTA == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
// Warp-converged variants: every lane of the (converged) warp executes the call with warp-uniform operands;
// elect.sync inside the asm picks the one lane that issues, so the compiler keeps descriptors in uniform
// registers instead of wrapping each instruction in an ELECT/R2UR.BROADCAST/BRA.U.ANY loop.
template <int NCTA>
__device__ __forceinline__ void umma_bf16_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  if constexpr (NCTA == 1) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
// One ring stage of the S GEMM in a single asm block (one elect for all of them): 4 MMAs over a 64-wide K box
// (descriptors advance by 32 B = 2 in the >>4 start-address field), plus 4 more over the second box of the
// stage at start offsets +AOFF / +BOFF when TWO_BOX.  The first MMA accumulates iff `accumulate`.  Operands
// are the low descriptor words of K-major SW128 tiles (start>>4 | LBO field); the high word is the constant
// SBO = 1024 B | version 1 | SWIZZLE_128B = 0x40004040, so only the low words are moved to uniform registers.
template <bool TWO_BOX, int AOFF, int BOFF>
__device__ __forceinline__ void umma_stage_pair(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t idesc,
                                                uint32_t accumulate) {
#define INFCL_MMA2(P) "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, " P ";\n\t"
#define INFCL_STEP(DA, DB) "add.u32 al, %1, " DA ";\n\tadd.u32 bl, %2, " DB ";\n\tmov.b64 a, {al, hi};\n\tmov.b64 b, {bl, hi};\n\t"
  if constexpr (TWO_BOX) {
    asm volatile(
        "{\n\t.reg .pred p, e, t;\n\t.reg .b64 a, b;\n\t.reg .b32 al, bl, hi;\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\tmov.b32 hi, 0x40004040;\n\t"
        INFCL_STEP("0", "0") INFCL_MMA2("p")
        INFCL_STEP("2", "2") INFCL_MMA2("t")
        INFCL_STEP("4", "4") INFCL_MMA2("t")
        INFCL_STEP("6", "6") INFCL_MMA2("t")
        INFCL_STEP("%5", "%6") INFCL_MMA2("t")
        INFCL_STEP("%7", "%8") INFCL_MMA2("t")
        INFCL_STEP("%9", "%10") INFCL_MMA2("t")
        INFCL_STEP("%11", "%12") INFCL_MMA2("t")
        "}" ::"r"(d_tmem), "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate),
        "n"(AOFF), "n"(BOFF), "n"(AOFF + 2), "n"(BOFF + 2), "n"(AOFF + 4), "n"(BOFF + 4), "n"(AOFF + 6), "n"(BOFF + 6)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e, t;\n\t.reg .b64 a, b;\n\t.reg .b32 al, bl, hi;\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\tmov.b32 hi, 0x40004040;\n\t"
        INFCL_STEP("0", "0") INFCL_MMA2("p")
        INFCL_STEP("2", "2") INFCL_MMA2("t")
        INFCL_STEP("4", "4") INFCL_MMA2("t")
        INFCL_STEP("6", "6") INFCL_MMA2("t")
        "}" ::"r"(d_tmem), "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate)
        : "memory");
  }
#undef INFCL_STEP
#undef INFCL_MMA2
}
// One ring stage of the backward's dA GEMM (dA^T += B_C^T G^T) in a single asm block: 8 MMAs over K = 128
// columns j; the MN-major A operand (B_C^T) advances by 16 rows of j = 2048 B (128 in the >>4 field) per MMA,
// the K-major B operand (G) by 32 B within its 64-column box and to the second box (+kBox = 512) after 4.
// Both descriptors have the high word 0x40004040 (SBO 1024 B, version 1, SWIZZLE_128B); the MN-major one
// carries LBO in its low word.  The first MMA accumulates iff `accumulate`.
template <int BOX2>
__device__ __forceinline__ void umma_stage_dA_pair(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t idesc,
                                                   uint32_t accumulate) {
#define INFCL_MMA2(P) "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, " P ";\n\t"
#define INFCL_STEP(DA, DB) "add.u32 al, %1, " DA ";\n\tadd.u32 bl, %2, " DB ";\n\tmov.b64 a, {al, hi};\n\tmov.b64 b, {bl, hi};\n\t"
  asm volatile(
      "{\n\t.reg .pred p, e, t;\n\t.reg .b64 a, b;\n\t.reg .b32 al, bl, hi;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\tmov.b32 hi, 0x40004040;\n\t"
      INFCL_STEP("0", "0") INFCL_MMA2("p")
      INFCL_STEP("128", "2") INFCL_MMA2("t")
      INFCL_STEP("256", "4") INFCL_MMA2("t")
      INFCL_STEP("384", "6") INFCL_MMA2("t")
      INFCL_STEP("512", "%5") INFCL_MMA2("t")
      INFCL_STEP("640", "%6") INFCL_MMA2("t")
      INFCL_STEP("768", "%7") INFCL_MMA2("t")
      INFCL_STEP("896", "%8") INFCL_MMA2("t")
      "}" ::"r"(d_tmem), "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate),
      "n"(BOX2), "n"(BOX2 + 2), "n"(BOX2 + 4), "n"(BOX2 + 6)
      : "memory");
#undef INFCL_STEP
#undef INFCL_MMA2
}
// One G tile x one 256-d chunk of the fused backward's dT GEMM (dT += G^T I, M = 256 columns j, N = 256 d, K = the
// tile's 128 rows i) in a single asm block: 8 MMAs of K = 16 rows, both operands MN-major.  A (G^T, j contiguous)
// lives in two 16-KB row halves (i 0-63, 64-127) of two 64-column boxes each: +2048 B (128 in the >>4 field) per
// MMA within a half, +16 KB (1024) after 4.  B (I, d contiguous) advances 16 rows = 2048 B per MMA.
__device__ __forceinline__ void umma_stage_dT_pair(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t idesc,
                                                   uint32_t accumulate) {
#define INFCL_MMA2(P) "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, " P ";\n\t"
#define INFCL_STEP(DA, DB) "add.u32 al, %1, " DA ";\n\tadd.u32 bl, %2, " DB ";\n\tmov.b64 a, {al, hi};\n\tmov.b64 b, {bl, hi};\n\t"
  asm volatile(
      "{\n\t.reg .pred p, e, t;\n\t.reg .b64 a, b;\n\t.reg .b32 al, bl, hi;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\tmov.b32 hi, 0x40004040;\n\t"
      INFCL_STEP("0", "0") INFCL_MMA2("p")
      INFCL_STEP("128", "128") INFCL_MMA2("t")
      INFCL_STEP("256", "256") INFCL_MMA2("t")
      INFCL_STEP("384", "384") INFCL_MMA2("t")
      INFCL_STEP("1024", "512") INFCL_MMA2("t")
      INFCL_STEP("1152", "640") INFCL_MMA2("t")
      INFCL_STEP("1280", "768") INFCL_MMA2("t")
      INFCL_STEP("1408", "896") INFCL_MMA2("t")
      "}" ::"r"(d_tmem), "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate)
      : "memory");
#undef INFCL_STEP
#undef INFCL_MMA2
}
// One G stage (128 columns j) x one 256-feature chunk of the 3-role backward's dI GEMM (dI += G B_C, M = 256 rows,
// N = 256 features, K = 128 j) in a single asm block: 8 MMAs of K = 16.  A (G, K-major, j contiguous) advances 32 B
// (2 in the >>4 field) within a 64-column box and jumps to the second box (+BOX2) after 4; B (B_C, MN-major,
// features contiguous) advances 16 rows = 2048 B (128) per MMA.
template <int BOX2>
__device__ __forceinline__ void umma_stage_kmn_pair(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t idesc,
                                                    uint32_t accumulate) {
#define INFCL_MMA2(P) "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, " P ";\n\t"
#define INFCL_STEP(DA, DB) "add.u32 al, %1, " DA ";\n\tadd.u32 bl, %2, " DB ";\n\tmov.b64 a, {al, hi};\n\tmov.b64 b, {bl, hi};\n\t"
  asm volatile(
      "{\n\t.reg .pred p, e, t;\n\t.reg .b64 a, b;\n\t.reg .b32 al, bl, hi;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\tmov.b32 hi, 0x40004040;\n\t"
      INFCL_STEP("0", "0") INFCL_MMA2("p")
      INFCL_STEP("2", "128") INFCL_MMA2("t")
      INFCL_STEP("4", "256") INFCL_MMA2("t")
      INFCL_STEP("6", "384") INFCL_MMA2("t")
      INFCL_STEP("%5", "512") INFCL_MMA2("t")
      INFCL_STEP("%6", "640") INFCL_MMA2("t")
      INFCL_STEP("%7", "768") INFCL_MMA2("t")
      INFCL_STEP("%8", "896") INFCL_MMA2("t")
      "}" ::"r"(d_tmem), "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate),
      "n"(BOX2), "n"(BOX2 + 2), "n"(BOX2 + 4), "n"(BOX2 + 6)
      : "memory");
#undef INFCL_STEP
#undef INFCL_MMA2
}
__device__ __forceinline__ void umma_commit_pair_mc_warp(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// commit all prior MMAs of this thread to an mbarrier (arrive::one when they complete)
__device__ __forceinline__ void umma_commit_1cta(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// pair version: arrive on the barrier at this offset in every CTA of `mask`
__device__ __forceinline__ void umma_commit_pair_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// ------------------------------------------------------------------ tcgen05: TMEM -> registers
// 32 lanes x 32 bit, 32 consecutive columns: thread t of the warp gets lane (base+t), columns [col, col+32)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 16 lanes x 256 bit, 8 repetitions along columns (16 lanes x 64 fp32 columns).  Thread t receives, for
// repetition rep (columns 8*rep .. 8*rep+7): v[rep*4 + 0,1] = lane (t/4), columns 8*rep + 2*(t%4) + {0,1};
// v[rep*4 + 2,3] = lane (t/4) + 8, same columns.  (CUTLASS Copy_Traits<SM100_TMEM_LOAD_16dp256b1x>.)
__device__ __forceinline__ void tmem_ld16x256x8(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ tcgen05: registers -> TMEM
// 32 lanes x 32 bit, 32 consecutive columns: thread t of the warp writes lane (base+t), columns [col, col+32)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ tcgen05: MMA with A in TMEM ("TS")
// D[tmem] (+)= A[tmem] * B[smem]^T, CTA pair.  For M = 128 (64 rows per CTA) the A operand uses the duplicated
// "2x2" data-path layout: lanes 0-31 and 64-95 both hold rows 0-31 of the CTA's 64, lanes 32-63 and 96-127 rows
// 32-63; a 32-bit column holds 2 consecutive K elements (bf16), K = 16 per MMA = 8 columns.
__device__ __forceinline__ void umma_ts_pair_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                  uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// One ring stage of the backward's dI GEMM in the TS form (dI += G B_C, M = 128 pair rows, N = 256 features, K = 128
// columns j) in a single asm block: 8 MMAs of K = 16; A (G, bf16 in TMEM) advances 8 columns per MMA, the MN-major B
// operand (B_C, features contiguous) 16 rows of j = 2048 B (128 in the >>4 field).  The first MMA accumulates iff
// `accumulate`.
__device__ __forceinline__ void umma_stage_dI_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t idesc,
                                                      uint32_t accumulate) {
#define INFCL_MMA2(P) "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [at], b, %3, " P ";\n\t"
#define INFCL_STEP(DA, DB) "add.u32 at, %1, " DA ";\n\tadd.u32 bl, %2, " DB ";\n\tmov.b64 b, {bl, hi};\n\t"
  asm volatile(
      "{\n\t.reg .pred p, e, t;\n\t.reg .b64 b;\n\t.reg .b32 at, bl, hi;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\tmov.b32 hi, 0x40004040;\n\t"
      INFCL_STEP("0", "0") INFCL_MMA2("p")
      INFCL_STEP("8", "128") INFCL_MMA2("t")
      INFCL_STEP("16", "256") INFCL_MMA2("t")
      INFCL_STEP("24", "384") INFCL_MMA2("t")
      INFCL_STEP("32", "512") INFCL_MMA2("t")
      INFCL_STEP("40", "640") INFCL_MMA2("t")
      INFCL_STEP("48", "768") INFCL_MMA2("t")
      INFCL_STEP("56", "896") INFCL_MMA2("t")
      "}" ::"r"(d_tmem), "r"(a_tmem), "r"(b_lo), "r"(idesc), "r"(accumulate)
      : "memory");
#undef INFCL_STEP
#undef INFCL_MMA2
}

// ------------------------------------------------------------------ descriptors
// Shared-memory matrix descriptor (sm_100 "version 1"): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), base_offset [49,52)=0, lbo_mode [52]=0, layout [61,64) (2 = SWIZZLE_128B).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptor, kind::f16: fp32 accumulate (c_format=1 at [4,6)), A=B=bf16 (format 1 at [7,10)
// and [10,13)), a_major [15], b_major [16] (0 = K-major, 1 = MN-major), N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ------------------------------------------------------------------ misc math
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {  // one FMNMX3 on sm_100
  float y;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(a), "f"(b), "f"(c));
  return y;
}
__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void red_add_v4_f32(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

}  // namespace infcl
