// tc_ptx.cuh -- thin inline-PTX wrappers for the sm_100a features the fused
// tensor-core kernel uses: mbarrier, TMA (cp.async.bulk.tensor), tcgen05
// (alloc / mma / commit / ld / fences) and shared-memory matrix descriptors.
// Bit layouts follow the PTX ISA (cross-checked against the CUTLASS headers
// shipped in this image: cute/arch/mma_sm100_desc.hpp, mma_sm100_umma.hpp).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hdc {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// HDC_MBAR_WAIT: 0 = try_wait (may suspend), 1 = test_wait spin, 2 = try_wait with a
// short suspend-time hint (HDC_MBAR_HINT_NS).
#ifndef HDC_MBAR_WAIT
#define HDC_MBAR_WAIT 0
#endif
#ifndef HDC_MBAR_HINT_NS
#define HDC_MBAR_HINT_NS 20
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
#if HDC_MBAR_WAIT == 1
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
#elif HDC_MBAR_WAIT == 2
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity), "n"(HDC_MBAR_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
#endif
}

// Spin (never suspends): for the latency-critical operand ring waits.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// Non-blocking probe: true iff the phase with parity `parity` has completed.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Bounded wait: true once the phase completed, false after ~`ns` nanoseconds (the thread
// may be suspended meanwhile instead of spinning on the barrier unit).
__device__ __forceinline__ bool mbar_try_wait_ns(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}

// Warp-uniform probe (lane 0 decides): keeps the MMA warp converged for elect.sync.
__device__ __forceinline__ bool mbar_test_uniform(uint64_t* bar, uint32_t parity) {
  return __shfl_sync(0xffffffffu, mbar_test(bar, parity) ? 1 : 0, 0) != 0;
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(desc) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* desc, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Multicast variant: the box lands at the same shared-memory offset in every CTA of
// `mask` (cluster ranks) and completes tx bytes on the mbarrier at `bar`'s offset in each.
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const void* desc, uint64_t* bar, int c0,
                                               int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// ---------------------------------------------------------------- clusters
// shared::cluster address of the same variable in CTA `cta` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(cta));
  return r;
}
// arrive on an mbarrier given by its shared::cluster address (possibly in a peer CTA)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(bytes)
               : "memory");
}
// 2-D TMA load into this CTA's shared memory whose completion is counted on the
// mbarrier at `bar_cluster` (shared::cluster address; the pair leader's barrier).
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const void* desc, uint32_t bar_cluster, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {  // every thread of every CTA of the cluster
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Orders this thread's generic-proxy shared-memory writes before later
// async-proxy (tensor core / TMA) reads of the same data.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_slot) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_slot) {  // warp 1 of both CTAs of a pair
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
               : "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Arrives on `bar` when all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, both K-major; one elected thread issues.
template <int KIND>  // 0: kind::f16 (bf16), 1: kind::tf32, 2: kind::i8
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  if constexpr (KIND == 0) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else if constexpr (KIND == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// Warp-collective variants: all 32 lanes execute, one elected lane issues.
// Keeping the MMA warp's control flow converged lets descriptors live in
// uniform registers (no per-MMA R2UR round trips from a divergent lane).
template <int KIND>
__device__ __forceinline__ void tc_mma_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  if constexpr (KIND == 0) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else if constexpr (KIND == 1) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
// One stage of Stage I in a single elected issue: 4 MMAs D (+)= A_k B_k^T (k = 0..3),
// the first accumulating iff `accumulate`.  One elect and all descriptors in uniform
// registers up front, so the four UTCHMMA issue back to back.
template <int KIND>
__device__ __forceinline__ void tc_mma4_elect(uint32_t d, uint64_t a0, uint64_t b0, uint64_t a1, uint64_t b1,
                                              uint64_t a2, uint64_t b2, uint64_t a3, uint64_t b3,
                                              uint32_t idesc, uint32_t accumulate) {
#define HDC_MMA4(KS)                                                                          \
  asm volatile(                                                                             \
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %10, 0;\n\t"   \
      "@e tcgen05.mma.cta_group::1." KS " [%0], %1, %2, %9, p;\n\t"                           \
      "@e tcgen05.mma.cta_group::1." KS " [%0], %3, %4, %9, 1;\n\t"                           \
      "@e tcgen05.mma.cta_group::1." KS " [%0], %5, %6, %9, 1;\n\t"                           \
      "@e tcgen05.mma.cta_group::1." KS " [%0], %7, %8, %9, 1;\n\t}" ::"r"(d),                \
      "l"(a0), "l"(b0), "l"(a1), "l"(b1), "l"(a2), "l"(b2), "l"(a3), "l"(b3), "r"(idesc),      \
      "r"(accumulate)                                                                          \
      : "memory")
  if constexpr (KIND == 0) HDC_MMA4("kind::f16");
  else if constexpr (KIND == 1) HDC_MMA4("kind::tf32");
  else HDC_MMA4("kind::i8");
#undef HDC_MMA4
}

template <int KIND>
__device__ __forceinline__ void tc_mma2_elect(uint32_t d, uint64_t a0, uint64_t b0, uint64_t a1, uint64_t b1,
                                              uint32_t idesc, uint32_t accumulate) {
#define HDC_MMA2(KS)                                                                          \
  asm volatile(                                                                             \
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %6, 0;\n\t"    \
      "@e tcgen05.mma.cta_group::1." KS " [%0], %1, %2, %5, p;\n\t"                           \
      "@e tcgen05.mma.cta_group::1." KS " [%0], %3, %4, %5, 1;\n\t}" ::"r"(d),                \
      "l"(a0), "l"(b0), "l"(a1), "l"(b1), "r"(idesc), "r"(accumulate)                          \
      : "memory")
  if constexpr (KIND == 0) HDC_MMA2("kind::f16");
  else if constexpr (KIND == 1) HDC_MMA2("kind::tf32");
  else HDC_MMA2("kind::i8");
#undef HDC_MMA2
}

// One int8 k-step of the 3-limb scheme (see k_fused_tc.cu): three MMAs, one elect.
__device__ __forceinline__ void tc_mma_i8x3_elect(uint32_t d0, uint64_t a0, uint64_t a1, uint64_t a2,
                                                  uint64_t b, uint32_t i240, uint32_t i160, uint32_t i80,
                                                  uint32_t dcol, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b32 d1, d2;\n\telect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\tadd.u32 d1, %0, %7;\n\tadd.u32 d2, d1, %7;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %4, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [d1], %2, %4, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [d2], %3, %4, %9, 1;\n\t}" ::"r"(d0),
      "l"(a0), "l"(a1), "l"(a2), "l"(b), "r"(i240), "r"(i160), "r"(dcol), "r"(accumulate), "r"(i80)
      : "memory");
}

// One int8 k-step of the wide mode (two 80-column sub-tiles s0, s1; see k_fused_tc.cu):
// TMEM accumulator blocks [A0s0 A0s1 A2s0 A2s1 A1s0 A1s1] and B row blocks
// [b0s0 b0s1 b2s0 b2s1 b1s0 b1s1], 80 columns / rows each, so the six limb products of both
// sub-tiles are five MMAs of N = 240, 240, 160, 160, 160 (an N <= 160 MMA costs as much as
// N = 160: tools/mma_microbench.cu):
//   x0 [b0s0 b0s1 b2s0] -> [A0s0 A0s1 A2s0]      x0 [b2s1 b1s0 b1s1] -> [A2s1 A1s0 A1s1]
//   x1 [b0s0 b0s1] -> [A1s0 A1s1]      x1 [b1s0 b1s1] -> [A2s0 A2s1]      x2 [b0s0 b0s1] -> [A2s0 A2s1]
// b0 / b3 / b4: descriptors of row blocks 0 / 3 / 4.
__device__ __forceinline__ void tc_mma_i8w5_elect(uint32_t d0, uint64_t a0, uint64_t a1, uint64_t a2,
                                                  uint64_t b0, uint64_t b3, uint64_t b4, uint32_t i240,
                                                  uint32_t i160, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b32 d1, d2, d3;\n\telect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %9, 0;\n\tadd.u32 d1, %0, 240;\n\tadd.u32 d2, %0, 320;\n\tadd.u32 d3, %0, 160;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %4, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [d1], %1, %5, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [d2], %2, %4, %8, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [d3], %2, %6, %8, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [d3], %3, %4, %8, 1;\n\t}" ::"r"(d0),
      "l"(a0), "l"(a1), "l"(a2), "l"(b0), "l"(b3), "l"(b4), "r"(i240), "r"(i160), "r"(accumulate)
      : "memory");
}

// CTA-pair (cta_group::2, M = 256) forms, issued by the leader CTA only: A rows 0-127
// from the leader's shared memory / TMEM lanes, 128-255 from the peer's; B's N extent
// split, the first half from the leader, the second from the peer (same offsets).
template <int KIND>
__device__ __forceinline__ void tc_mma4_pair_elect(uint32_t d, uint64_t a0, uint64_t b0, uint64_t a1, uint64_t b1,
                                                   uint64_t a2, uint64_t b2, uint64_t a3, uint64_t b3,
                                                   uint32_t idesc, uint32_t accumulate) {
#define HDC_MMA4P(KS)                                                                         \
  asm volatile(                                                                             \
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %10, 0;\n\t"   \
      "@e tcgen05.mma.cta_group::2." KS " [%0], %1, %2, %9, p;\n\t"                           \
      "@e tcgen05.mma.cta_group::2." KS " [%0], %3, %4, %9, 1;\n\t"                           \
      "@e tcgen05.mma.cta_group::2." KS " [%0], %5, %6, %9, 1;\n\t"                           \
      "@e tcgen05.mma.cta_group::2." KS " [%0], %7, %8, %9, 1;\n\t}" ::"r"(d),                \
      "l"(a0), "l"(b0), "l"(a1), "l"(b1), "l"(a2), "l"(b2), "l"(a3), "l"(b3), "r"(idesc),      \
      "r"(accumulate)                                                                          \
      : "memory")
  if constexpr (KIND == 0) HDC_MMA4P("kind::f16");
  else HDC_MMA4P("kind::tf32");
#undef HDC_MMA4P
}
__device__ __forceinline__ void tc_mma_ts_pair_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                                     uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair_mc_elect(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// A operand from TMEM (kind::f16, K-major: lane = row, 2 bf16 per 32-bit column,
// element k of a K=16 step at column k/2, low half for even k), B from shared memory.
__device__ __forceinline__ void tc_mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Commit arriving on the mbarrier at `bar`'s offset in every CTA of `mask`.
__device__ __forceinline__ void tc_commit_mc_elect(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// 32 lanes x 32-bit, 8 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}
// 32 lanes x 32-bit, 4 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
// 32 lanes x 32-bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 32 lanes x 32-bit stores, 8 consecutive columns per thread (registers -> TMEM).
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&r)[8]) {  // r[0..3]
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor, K-major, SWIZZLE_64B canonical layout:
// rows of 64 bytes, 8-row core groups 512 B apart (SBO), LBO unused (16 B).
// Fields: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version=1 [46,48),
// base_offset=0 [49,52), lbo_mode=0 [52], layout_type [61,64) (SW64 = 4).
__device__ __forceinline__ uint64_t smem_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

// K-major swizzled layout (layout_type 2 = SWIZZLE_128B, 4 = SWIZZLE_64B): rows of
// the atom width, 8-row groups `sbo` bytes apart.
__device__ __forceinline__ uint64_t smem_desc_sw(uint32_t saddr, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// K-major, no swizzle ("interleaved"): 8-row x 16-byte core matrices; LBO =
// byte distance between K-adjacent core matrices, SBO = between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc_interleaved(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;  // layout_type 0 = SWIZZLE_NONE
}

// Instruction descriptor (kind::f16 / tf32 / i8), both operands K-major.
// c_format [4,6): 1 = F32, 2 = S32; a/b_format [7,10)/[10,13): bf16 = 1,
// tf32 = 2, signed int8 = 1; n_dim [17,23) = N >> 3; m_dim [24,29) = M >> 4.
template <int KIND>
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  const uint32_t cfmt = (KIND == 2) ? 2u : 1u;
  const uint32_t abfmt = (KIND == 0) ? 1u : (KIND == 1) ? 2u : 1u;
  return (cfmt << 4) | (abfmt << 7) | (abfmt << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

}  // namespace ptx
}  // namespace hdc
