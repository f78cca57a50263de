// ptx_sm100.cuh — thin inline-PTX wrappers for the sm_100a features the
// attention kernel uses: mbarriers, TMA tensor loads, tcgen05 (TMEM alloc,
// MMA, commit, ld/st, fences) and UMMA shared-memory / instruction
// descriptors. No CuTe/CUTLASS dependency; encodings follow the PTX ISA for
// sm_100a (descriptor bit layout cross-checked against the vendored CuTe
// headers' SmemDescriptor / InstrDescriptor unions).
#pragma once

#include <cstdint>

namespace uspb200 {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// One lane of a converged warp (elect.sync); the others get false.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar_addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar_addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Blocks until the phase with the given parity has completed.
// A pipeline deadlock traps (the launch fails with an error) instead of
// hanging the GPU; the bound is far beyond any legitimate wait.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t spins = 0;
  while (!mbar_try_wait(a, parity)) {
    if (++spins == (1u << 28)) __trap();
  }
}

// Explicit shared-space accesses (a pointer derived from the aligned
// dynamic-smem base is generic to the compiler; LD.E/ST.E on it cost a
// long-scoreboard round trip each).
__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// --------------------------------------------------------------- clusters
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cta address -> the shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t bar_addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar_addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t spins = 0;
  while (!mbar_try_wait_cluster(a, parity)) {
    if (++spins == (1u << 28)) __trap();
  }
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// --------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// 4-D tiled load global -> shared, completion signalled on `bar` (tx bytes).
__device__ __forceinline__ void tma_load_4d(void* dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3)
      : "memory");
}
// TMA reduction shared -> global: the box at {c0..c3} of the fp32 tensor
// behind `tmap` += the dense box in shared memory (bulk_group completion).
__device__ __forceinline__ void tma_reduce_add_4d(const void* tmap, const void* src, int c0, int c1, int c2,
                                                  int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group"
      " [%0, {%2, %3, %4, %5}], [%1];" ::"l"(reinterpret_cast<uint64_t>(tmap)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Waits until at most N committed bulk groups still READ their shared source.
template <int N>
__device__ __forceinline__ void bulk_wait_group_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_group() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// Plain bulk copy global -> shared (16-byte multiple), completion on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// The same load multicast to every CTA of the cluster in `mask`: data and
// complete_tx land at the same shared-memory offsets in each of them.
__device__ __forceinline__ void tma_load_4d_mc(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2,
                                               int c3, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "h"(mask)
      : "memory");
}
// A CTA pair's load: data into this CTA's shared memory, completion signalled
// on the barrier at `mbar_cluster` (a shared::cluster address, the leader's).
__device__ __forceinline__ void tma_load_4d_2sm(void* dst, const void* tmap, uint32_t mbar_cluster, int c0, int c1,
                                                int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(mbar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_hint(void* dst, const void* tmap, uint64_t* bar, int c0,
                                                 int c1, int c2, int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ----------------------------------------------------------------- tcgen05
// Warp-collective TMEM allocation; the base address is written to *dst.
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
// cta_group::2: the same warp of both CTAs of a pair allocates; the two
// allocations are at the same TMEM address.
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate).
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem].
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// ---- batched MMA issue: one asm block per K/V tile and Q tile, so the
// compiler converts the operands to uniform registers once per block
// instead of once per instruction (issue overhead was the MMA warp's limit).
// S[128 x 128] (+)= Q[128 x HS] K[128 x HS]^T over HS/16 k-steps. Descriptors
// advance 32 B inside a 128-byte swizzle row and 16 KB to the next 64-column
// block (units of 16 bytes in the descriptor's start-address field).
__device__ __forceinline__ void mma_qk_hs128(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p0, p1;\n\t.reg .b64 ra, rb;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.u32 p1, 1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p0;\n\t"
      "add.s64 ra, %1, 2;\n\tadd.s64 rb, %2, 2;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 4;\n\tadd.s64 rb, %2, 4;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 6;\n\tadd.s64 rb, %2, 6;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1024;\n\tadd.s64 rb, %2, 1024;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1026;\n\tadd.s64 rb, %2, 1026;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1028;\n\tadd.s64 rb, %2, 1028;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1030;\n\tadd.s64 rb, %2, 1030;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_qk_hs64(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p0, p1;\n\t.reg .b64 ra, rb;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.u32 p1, 1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p0;\n\t"
      "add.s64 ra, %1, 2;\n\tadd.s64 rb, %2, 2;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 4;\n\tadd.s64 rb, %2, 4;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 6;\n\tadd.s64 rb, %2, 6;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// cta_group::2 (M = 256 over a CTA pair): S = Q K^T with each CTA's own
// 128 Q rows (A, 16 KB column blocks) and ITS HALF of the K tile (B: 64 key
// rows, 8 KB column blocks); issued by the leader CTA only.
__device__ __forceinline__ void mma2_qk_hs128(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p0, p1;\n\t.reg .b64 ra, rb;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.u32 p1, 1, 1;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p0;\n\t"
      "add.s64 ra, %1, 2;\n\tadd.s64 rb, %2, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 4;\n\tadd.s64 rb, %2, 4;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 6;\n\tadd.s64 rb, %2, 6;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1024;\n\tadd.s64 rb, %2, 512;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1026;\n\tadd.s64 rb, %2, 514;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1028;\n\tadd.s64 rb, %2, 516;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1030;\n\tadd.s64 rb, %2, 518;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// O += P V over a CTA pair: P from each CTA's TMEM, V's 64-column half of
// each CTA (B, N split across the pair); leader only.
__device__ __forceinline__ void mma2_pv_chain(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p0, p1;\n\t.reg .b64 rb;\n\t.reg .b32 ta;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.u32 p1, 1, 1;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p0;\n\t"
      "add.u32 ta, %1, 8;\n\tadd.s64 rb, %2, 128;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 16;\n\tadd.s64 rb, %2, 256;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 24;\n\tadd.s64 rb, %2, 384;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 32;\n\tadd.s64 rb, %2, 512;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 40;\n\tadd.s64 rb, %2, 640;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 48;\n\tadd.s64 rb, %2, 768;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 56;\n\tadd.s64 rb, %2, 896;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma2_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// O[128 x N] (+)= P[128 x 128] V[128 x N]: P (bf16) from TMEM, 8 columns per
// 16-key step; V MN-major, 16 rows (2 KB) per step.
__device__ __forceinline__ void mma_pv_chain(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p0, p1;\n\t.reg .b64 rb;\n\t.reg .b32 ta;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.u32 p1, 1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n\t"
      "add.u32 ta, %1, 8;\n\tadd.s64 rb, %2, 128;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 16;\n\tadd.s64 rb, %2, 256;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 24;\n\tadd.s64 rb, %2, 384;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 32;\n\tadd.s64 rb, %2, 512;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 40;\n\tadd.s64 rb, %2, 640;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 48;\n\tadd.s64 rb, %2, 768;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "add.u32 ta, %1, 56;\n\tadd.s64 rb, %2, 896;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Two consecutive 16-deep k-steps of a TS MMA: A from TMEM columns a, a+8
// (bf16 packed), B MN-major 16 rows (2 KB) further per step.
__device__ __forceinline__ void mma_ts_k2(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p0, p1;\n\t.reg .b64 rb;\n\t.reg .b32 ta;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.u32 p1, 1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n\t"
      "add.u32 ta, %1, 8;\n\tadd.s64 rb, %2, 128;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], rb, %3, p1;\n\t"
      "}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[128 x N] (+)= A[128 x 128] B[128 x N], both from shared memory, 8
// k-steps of 16: A K-major (32 B per step inside a 128-byte swizzle row,
// 16 KB to the next 64-column block), B MN-major (16 rows = 2 KB per step).
// The fused backward's dK += dS^T Q (A = dS^T as the compute warps stored it).
__device__ __forceinline__ void mma_kmaj_mn_chain(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p0, p1;\n\t.reg .b64 ra, rb;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.u32 p1, 1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p0;\n\t"
      "add.s64 ra, %1, 2;\n\tadd.s64 rb, %2, 128;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 4;\n\tadd.s64 rb, %2, 256;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 6;\n\tadd.s64 rb, %2, 384;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1024;\n\tadd.s64 rb, %2, 512;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1026;\n\tadd.s64 rb, %2, 640;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1028;\n\tadd.s64 rb, %2, 768;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 1030;\n\tadd.s64 rb, %2, 896;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[128 x N] (+)= A[128 x 128] B[128 x N] with BOTH operands MN-major in
// shared memory (16 rows = 2 KB per k-step each): the fused backward's
// dQ^T = K^T dS^T (A = the K tile, B = dS^T, both stored key-row-major).
__device__ __forceinline__ void mma_mn_mn_chain(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p0, p1;\n\t.reg .b64 ra, rb;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\t"
      "setp.eq.u32 p1, 1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p0;\n\t"
      "add.s64 ra, %1, 128;\n\tadd.s64 rb, %2, 128;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 256;\n\tadd.s64 rb, %2, 256;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 384;\n\tadd.s64 rb, %2, 384;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 512;\n\tadd.s64 rb, %2, 512;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 640;\n\tadd.s64 rb, %2, 640;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 768;\n\tadd.s64 rb, %2, 768;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "add.s64 ra, %1, 896;\n\tadd.s64 rb, %2, 896;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p1;\n\t"
      "}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrives on `bar` once every previously issued tcgen05 op of this thread has
// completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Commit arriving on the barrier at this offset in every CTA of `mask`.
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

#define USPB_R8(a, o) a[o + 0], a[o + 1], a[o + 2], a[o + 3], a[o + 4], a[o + 5], a[o + 6], a[o + 7]
#define USPB_W8(a, o)                                                                         \
  "=r"(a[o + 0]), "=r"(a[o + 1]), "=r"(a[o + 2]), "=r"(a[o + 3]), "=r"(a[o + 4]),           \
      "=r"(a[o + 5]), "=r"(a[o + 6]), "=r"(a[o + 7])
#define USPB_RW8(a, o)                                                                        \
  "+r"(a[o + 0]), "+r"(a[o + 1]), "+r"(a[o + 2]), "+r"(a[o + 3]), "+r"(a[o + 4]),           \
      "+r"(a[o + 5]), "+r"(a[o + 6]), "+r"(a[o + 7])
#define USPB_IN8(a, o)                                                                        \
  "r"(a[o + 0]), "r"(a[o + 1]), "r"(a[o + 2]), "r"(a[o + 3]), "r"(a[o + 4]), "r"(a[o + 5]), \
      "r"(a[o + 6]), "r"(a[o + 7])

// 32 lanes x 32 consecutive 32-bit columns: thread i gets lane (base+i).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : USPB_W8(r, 0), USPB_W8(r, 8), USPB_W8(r, 16), USPB_W8(r, 24)
      : "r"(taddr)
      : "memory");
}
// Waits for outstanding tcgen05.ld; the "+r" ties keep consumers of r after it.
__device__ __forceinline__ void tmem_ld_wait(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : USPB_RW8(r, 0), USPB_RW8(r, 8), USPB_RW8(r, 16), USPB_RW8(r, 24)
               :
               : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      USPB_IN8(r, 0), USPB_IN8(r, 8), USPB_IN8(r, 16), USPB_IN8(r, 24)
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// --------------------------------------------------------- UMMA descriptors
// Shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), version 1.
//   bits [0,14) start>>4, [16,30) LBO>>4, [32,46) SBO>>4, [46,48) version,
//   [49,52) base offset (0: operands are 1024B aligned), [61,64) layout.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

// Instruction descriptor, kind::f16: bf16 A/B, fp32 D.
//   [4,6) D fmt (1=f32), [7,10) A fmt (1=bf16), [10,13) B fmt (1=bf16),
//   [15] A major (0=K), [16] B major (1=MN), [17,23) N>>3, [24,29) M>>4.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N, uint32_t a_mn,
                                                      uint32_t b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}

// ------------------------------------------------------------------- math
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2): one issue slot per pair.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\t"
      "mov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
      "mov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\t"
      "mov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\t"
      "mov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\t"
      "mov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\t"
      "mov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fadd2_rm(float2 a, float2 b) {  // rounded toward -inf
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\t"
      "mov.b64 rb, {%4, %5};\n\t"
      "add.rm.f32x2 rd, ra, rb;\n\t"
      "mov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// 2^x for a pair on the FMA pipe (x <= 126): 2^x = 2^floor(x) * p(f),
// f = x - floor(x) in [0, 1), p a degree-3 polynomial with p(0) = 1 exactly
// (max rel. error 8.8e-5, below bf16's 3.9e-3). x is clamped at -127, where
// f = 0 and the exponent arithmetic gives exactly +0 — what ex2.approx.ftz
// returns for masked (-inf) scores. Offloads a fraction of the softmax
// exponentials from the 16/clk/SM MUFU unit.
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 t = fadd2_rm(x, magic);                        // floor(x) in the low mantissa bits
  const float2 j = fadd2(t, make_float2(-12582912.f, -12582912.f));  // floor(x), exact
  const float2 f = ffma2(j, make_float2(-1.f, -1.f), x);             // x - floor(x), exact
  float2 p = ffma2(make_float2(0.077119089663028717f, 0.077119089663028717f), f,
                   make_float2(0.227564394474029541f, 0.227564394474029541f));
  p = ffma2(p, f, make_float2(0.695146143436431885f, 0.695146143436431885f));
  p = ffma2(p, f, make_float2(1.f, 1.f));
  const uint32_t bx = __float_as_uint(p.x) + (__float_as_uint(t.x) << 23);
  const uint32_t by = __float_as_uint(p.y) + (__float_as_uint(t.y) << 23);
  return make_float2(__uint_as_float(bx), __uint_as_float(by));
}
// bf16x2 packing of two NON-NEGATIVE finite floats on the integer pipes:
// round half up (+0x8000 on the bit pattern; differs from RNE only at exact
// ties) and keep the high halves with one PRMT. cvt.rn.bf16x2.f32 (F2FP)
// issues on the same 16-lane/clk/SM pipe as MUFU.EX2, so in the softmax it
// would compete with the exponentials.
__device__ __forceinline__ uint32_t pack_bf16x2_pos(float lo, float hi) {
  const uint32_t a = __float_as_uint(lo) + 0x8000u;
  const uint32_t b = __float_as_uint(hi) + 0x8000u;
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// The same integer-pipe packing for finite floats of either sign: the bit
// pattern is sign-magnitude, so +0x8000 rounds |x| half up (ties away from
// zero instead of to even). Used for dS in the backward, where
// cvt.rn.bf16x2.f32 would double the load on the MUFU pipe the exponentials
// already saturate.
__device__ __forceinline__ uint32_t pack_bf16x2_int(float lo, float hi) { return pack_bf16x2_pos(lo, hi); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

}  // namespace ptx
}  // namespace uspb200
