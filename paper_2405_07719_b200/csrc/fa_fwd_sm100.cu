// fa_fwd_sm100.cu — per-block flash-attention forward for sm_100a.
//
// The B200 restatement of SoftmaxState::update / finalize / logsumexp
// (reference src/numerics/attention.cpp:181-264), one launch per ring step
// (src/usp/ring_attention.cpp:62-75). Design:
//
//   * persistent CTAs, one per SM, walking a host-built LPT-ordered list of
//     work units (batch, q-head pair, 128-row query tile);
//   * warp-specialised: 1 TMA producer warp, 1 MMA-issuer warp (one elected
//     thread issues every tcgen05.mma), 4*NQ softmax warps (one TMEM lane =
//     one query row per thread);
//   * NQ = 2 query tiles per CTA = two q heads of the same GQA group over the
//     same rows, so every K/V tile staged in shared memory feeds both, and
//     the tensor core alternates between the tiles while the other's
//     softmax runs (one shared S, P_A, P_B, O_A, O_B fill the 512 TMEM
//     columns at head size 128);
//   * S = Q K^T: tcgen05.mma SS (Q, K from 128B-swizzled smem via TMA) into
//     TMEM; P = exp2(S*scale*log2e - m) is written back over S as bf16 and
//     O += P V runs as a TS MMA (P from TMEM, V MN-major from smem);
//   * O is rescaled lazily: the running max only moves when it grows by more
//     than 2^8, so the TMEM read-modify-write of O is rare;
//   * the epilogue normalises, merges into the fp32 ring-step running state
//     (log-sum-exp merge) and/or writes bf16 O + natural-log LSE.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "fa_fwd.hpp"
#include "ptx_sm100.cuh"

#ifndef USPB_FWD_SPLITLD
#define USPB_FWD_SPLITLD 1  // S read from TMEM in two halves (A/B: tools/ab_fwd.py)
#endif
#ifndef USPB_FWD_POLY64
#define USPB_FWD_POLY64 2  // head size 64: exponential pairs of every 8 computed on the FMA pipe
#endif
#ifndef USPB_FWD_STAGES
#define USPB_FWD_STAGES 4  // K/V pipeline depth: measured best at 4 (2 tiles of K+V) on B200
#endif
namespace uspb200 {

using namespace ptx;

template <int NQ, int HS>
struct FwdCfg {
  static constexpr int kCols = 128;  // key columns per softmax thread (one TMEM lane = one query row)
  static constexpr int kSoftmaxWarps = 4 * NQ;
  static constexpr int kTmaWarp = kSoftmaxWarps;
  static constexpr int kMmaWarp = kSoftmaxWarps + 1;
  // NQ == 2: a full extra warpgroup (TMA, MMA, 2 idle warps) so registers
  // can be moved to the softmax warpgroups with setmaxnreg.
  static constexpr bool kRegSplit = NQ == 2;
  // producer warpgroup: TMA warp, S-issue warp, PV-issue warp, 1 idle
  static constexpr int kPvWarp = kSoftmaxWarps + 2;
  static constexpr int kThreads = 32 * (kSoftmaxWarps + 4);
  // setmaxnreg only redistributes the registers allocated at launch
  // (kThreads x kLaunchRegs under __launch_bounds__(kThreads, 1)); asking for
  // more would block the .inc forever.
  static constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8;
  static constexpr int kProducerRegs = 88;
  static constexpr int kSoftmaxRegs =
      ((kLaunchRegs * kThreads - 128 * kProducerRegs) / (32 * kSoftmaxWarps)) / 8 * 8 > 240
          ? 240
          : ((kLaunchRegs * kThreads - 128 * kProducerRegs) / (32 * kSoftmaxWarps)) / 8 * 8;
  static_assert(!kRegSplit || 32 * kSoftmaxWarps * kSoftmaxRegs + 128 * kProducerRegs <= kThreads * kLaunchRegs,
                "register split exceeds the launch allocation");
  static constexpr int kSub = HS / 64;           // 128-byte (64 x bf16) column blocks
  static constexpr int kSubBytes = 128 * 128;    // one block: 128 rows x 128 B
  static constexpr int kQBytes = kTileM * HS * 2;
  static constexpr int kKVBytes = kTileN * HS * 2;
  static constexpr int kBudget = 227 * 1024 - 2048;
  static constexpr int kStagesFit = (kBudget - NQ * kQBytes) / kKVBytes;
  static constexpr int kStages = kStagesFit > USPB_FWD_STAGES ? USPB_FWD_STAGES : kStagesFit;
  static constexpr int kSchedDepth = 4;  // unit-ticket ring between producer and consumers
  static constexpr int kNumBars = 3 * NQ + 2 + NQ + 2 * kStages + 2 * kSchedDepth;
  static constexpr int kSmemBytes = 1024 /*align slack*/ + NQ * kQBytes + kStages * kKVBytes +
                                    kNumBars * 8 + 16 + 4 * kSchedDepth;
  // TMEM: ONE S buffer shared by the q tiles (time-multiplexed: the MMA
  // warp computes the next tile's S as soon as the previous S has been
  // loaded into registers), a private P (bf16, 64 columns) and O per q tile.
  static constexpr uint32_t kSCol = 0;                   // S: 128 fp32 columns
  static constexpr uint32_t kPCol = 128;                 // P_t at kPCol + 64*t
  static constexpr uint32_t kOCol = 128 + 64 * NQ;       // O_t at kOCol + HS*t
  static constexpr uint32_t kColsUsed = kOCol + NQ * HS;
  static constexpr uint32_t kTmemCols = kColsUsed <= 128 ? 128 : (kColsUsed <= 256 ? 256 : 512);
  static_assert(HS == 64 || HS == 128, "head_size must be 64 or 128 on the tcgen05 path");
  static_assert(kStages >= 2, "not enough shared memory for a K/V pipeline");
};

// Development trace: event ev of tile i, CTA 0 only. Compiled in only with
// -DUSPB_TRACE (tools/trace_fa.py builds that variant); the production
// kernel carries no instrumentation (it costs issue slots and I-cache).
// `dep` orders the clock read after the value it depends on.
__device__ __forceinline__ void trace_ev(const FwdParams& p, int ev, uint32_t i, float dep = 0.f) {
#ifndef USPB_TRACE
  (void)p, (void)ev, (void)i, (void)dep;
  return;
#endif
  if (p.trace != nullptr && blockIdx.x == 0 && i < static_cast<uint32_t>(kTraceTiles)) {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) : "f"(dep));
    p.trace[ev * kTraceTiles + i] = c;
  }
}

// tcgen05.commit from one elected lane of a converged warp.
__device__ __forceinline__ void commit_one(uint64_t* bar) {
  if (elect_one()) mma_commit(bar);
  __syncwarp();
}

// Calls f(integral_constant<int, S>) with S == slot (slot < N): turns a
// runtime pipeline-stage index into a compile-time smem offset.
template <int N, class F>
__device__ __forceinline__ void dispatch_slot(uint32_t slot, F&& f) {
  if constexpr (N > 0) {
    if (slot == N - 1)
      f(std::integral_constant<int, N - 1>{});
    else
      dispatch_slot<N - 1>(slot, f);
  }
}

// Consumer side of the unit-ticket ring: every consumer warp waits for slot
// it % depth, reads the unit index, and one lane per warp releases the slot.
// whole_warp: all 32 lanes run this (softmax warps); otherwise a single
// lane (the MMA issuer) does.
// MC (2-CTA cluster): the tickets are written by the leader CTA into both
// CTAs' slots and every consumer releases the LEADER's slot.
template <int kDepth, int MC>
__device__ __forceinline__ int next_unit_impl(uint64_t* full, uint64_t* empty, const int* slot,
                                              uint32_t it, bool whole_warp) {
  const uint32_t d = it % kDepth;
  if constexpr (MC)
    mbar_wait_cluster(&full[d], (it / kDepth) & 1);
  else
    mbar_wait(&full[d], (it / kDepth) & 1);
  const int u = *reinterpret_cast<const volatile int*>(&slot[d]);
  if (whole_warp) __syncwarp();
  if (!whole_warp || lane_id() == 0) {
    if constexpr (MC)
      mbar_arrive_cluster(mapa_shared(smem_u32(&empty[d]), 0));
    else
      mbar_arrive(&empty[d]);
  }
  return u;
}
#define next_unit(full, empty, slot, it, whole_warp) \
  next_unit_impl<C::kSchedDepth, MC>(full, empty, slot, it, whole_warp)

// MC = 1: a 2-CTA cluster runs the two head pairs of a 4-head GQA group over
// the same rows (unit = q tile x head quad); each CTA loads half of every
// K/V tile and multicasts it to both, so L2->SMEM traffic per FLOP halves.
template <int NQ, int HS, int MC>
__global__ void __launch_bounds__(FwdCfg<NQ, HS>::kThreads, 1)
    fa_fwd_sm100_kernel(const __grid_constant__ FwdParams p) {
  using C = FwdCfg<NQ, HS>;
  static_assert(!MC || (NQ == 2 && HS == 128), "cluster mode: two head pairs, 128-column tiles");
  // MC == 2: cta_group::2 MMAs (M = 256 over the pair): the leader CTA issues
  // every MMA; each CTA holds its own Q tiles, one 64-key half of every K
  // tile and one 64-column half of every V tile.
  constexpr bool k2 = MC == 2;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + NQ * C::kQBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + NS * C::kKVBytes);
  uint64_t* q_full = bars;              // [NQ]  TMA -> MMA
  uint64_t* q_empty = q_full + NQ;      // [1]   MMA -> TMA
  uint64_t* kv_full = q_empty + 1;      // [NS]  TMA -> MMA
  uint64_t* kv_empty = kv_full + NS;    // [NS]  MMA -> TMA
  uint64_t* s_full = kv_empty + NS;     // [NQ]  MMA -> softmax
  uint64_t* p_ready = s_full + NQ;      // [NQ]  softmax -> MMA (128 arrivals)
  uint64_t* pv_done = p_ready + NQ;     // [NQ]  MMA -> softmax: PV_t finished (P_t, O_t free)
  uint64_t* s_free = pv_done + NQ;      // [1]   softmax -> MMA: the S buffer was loaded
  uint64_t* sched_full = s_free + 1;            // [D] producer -> consumers
  uint64_t* sched_empty = sched_full + C::kSchedDepth;  // [D] consumers -> producer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched_empty + C::kSchedDepth);
  int* sched_slot = reinterpret_cast<int*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = MC ? cluster_ctarank() : 0u;
  // the head pair a unit's hp field names for this CTA
  auto unit_hp = [&](uint32_t unit) { return MC ? int((unit >> 16) & 0xFF) * 2 + int(crank) : int((unit >> 16) & 0xFF); };

  if (threadIdx.x == 0) {
    for (int t = 0; t < NQ; ++t) {
      mbar_init(&q_full[t], 1);
      mbar_init(&s_full[t], 1);
      mbar_init(&p_ready[t], k2 ? 2 * 4 : 128);  // 2SM: one lane per warp of both CTAs
      mbar_init(&pv_done[t], 1);
    }
    mbar_init(s_free, (k2 ? 2 : 1) * 4);  // one lane of each warp holding S (both CTAs with 2SM)
    mbar_init(q_empty, 1);
    for (int d = 0; d < C::kSchedDepth; ++d) {
      mbar_init(&sched_full[d], 1);
      // S warp, PV warp, softmax warps (of both CTAs + the peer's TMA warp with MC)
      mbar_init(&sched_empty[d], MC ? 2 * (2 + C::kSoftmaxWarps) + 1 : 2 + C::kSoftmaxWarps);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], MC == 1 ? 2 : 1);  // MC 1: both CTAs' MMAs have read the slot
    }
    fence_barrier_init();
  }
  if (warp == C::kMmaWarp) {
    if constexpr (k2)
      tmem_alloc_2sm(tmem_slot, C::kTmemCols);
    else
      tmem_alloc(tmem_slot, C::kTmemCols);
  }
  if (warp == C::kTmaWarp && lane == 0) {
    tma_prefetch_desc(&p.tm_q);
    tma_prefetch_desc(&p.tm_k);
    tma_prefetch_desc(&p.tm_v);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC > 0) cluster_sync();  // the peer's barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // One CTA per SM (shared memory) owns all of TMEM, so the allocation
  // starts at lane 0 / column 0; the MMA issue relies on that.
  if (tmem != 0) __trap();
  const int group = p.heads / p.kv_heads;  // q heads per kv head (GQA)

  if (warp < C::kSoftmaxWarps) {
    // ------------------------------------------------------------ softmax
    if constexpr (C::kRegSplit)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::kSoftmaxRegs));
    constexpr int KC = C::kCols;
    const int t = warp / 4;
    const int quarter = warp & 3;             // TMEM lane quarter (warp id % 4)
    const int row_in_tile = quarter * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t s_addr = lane_base + C::kSCol;
    const uint32_t p_addr = lane_base + C::kPCol + t * 64;
    const uint32_t o_addr = lane_base + C::kOCol + t * HS;
    const float sl2 = p.scale_log2;
    uint32_t s_phase = 0, pv_phase = 0;
    for (uint32_t it = 0;; ++it) {
      const int u = next_unit(sched_full, sched_empty, sched_slot, it, true);
      if (u >= p.num_units) break;
      const uint32_t unit = p.units[u];
      const int qt = unit & 0xFFFF, hp = unit_hp(unit), b = unit >> 24;
      const int h = p.pair_rows ? hp : hp * NQ + t;
      const int beg = p.tile_off[qt];
      const int n = p.tile_off[qt + 1] - beg;
      const int q_row = (p.pair_rows ? qt * NQ + t : qt) * kTileM + row_in_tile;
      const int qpos = p.q_pos[q_row];
      // running max m_run (log2 units, of S * scale * log2 e); P = 2^(s - m_run)
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n; ++j) {
        const int entry = p.tile_list[beg + j];
        if constexpr (k2)
          mbar_wait_cluster(&s_full[t], s_phase & 1);
        else
          mbar_wait(&s_full[t], s_phase & 1);
        const bool tr = quarter == 0 && lane == 0;
        if (tr) trace_ev(p, 0 + 5 * t, s_phase);
        ++s_phase;
        tc_fence_after();
        uint32_t s[KC];
#if USPB_FWD_SPLITLD
        // Two halves: the first half's mask and max run under the second
        // half's TMEM load latency.
        constexpr int KH = KC / 2;
#pragma unroll
        for (int c = 0; c < KH / 32; ++c) tmem_ld32(s_addr + c * 32, s + c * 32);
#pragma unroll
        for (int c = 0; c < KH / 32; ++c) tmem_ld_wait(s + c * 32);
#pragma unroll
        for (int c = KH / 32; c < KC / 32; ++c) tmem_ld32(s_addr + c * 32, s + c * 32);
        const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + (entry & 0x7FFFFFFF) * kTileN);
        auto mask4 = [&](int c) {  // partial tile: the position mask per element
          const int4 kp = __ldg(kp4 + c);
          if (kp.x > qpos) s[4 * c + 0] = __float_as_uint(-INFINITY);
          if (kp.y > qpos) s[4 * c + 1] = __float_as_uint(-INFINITY);
          if (kp.z > qpos) s[4 * c + 2] = __float_as_uint(-INFINITY);
          if (kp.w > qpos) s[4 * c + 3] = __float_as_uint(-INFINITY);
        };
        if (entry < 0) {
#pragma unroll
          for (int c = 0; c < KH / 4; ++c) mask4(c);
        }
        float mx0 = __uint_as_float(s[0]), mx1 = __uint_as_float(s[1]);
        float mx2 = __uint_as_float(s[2]), mx3 = __uint_as_float(s[3]);
#pragma unroll
        for (int i = 4; i < KH; i += 4) {
          mx0 = fmaxf(mx0, __uint_as_float(s[i + 0]));
          mx1 = fmaxf(mx1, __uint_as_float(s[i + 1]));
          mx2 = fmaxf(mx2, __uint_as_float(s[i + 2]));
          mx3 = fmaxf(mx3, __uint_as_float(s[i + 3]));
        }
#pragma unroll
        for (int c = KH / 32; c < KC / 32; ++c) tmem_ld_wait(s + c * 32);
        // S is in registers: the shared S buffer may take the next S.
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (k2)
            mbar_arrive_cluster(mapa_shared(smem_u32(s_free), 0));
          else
            mbar_arrive(s_free);
        }
        if (tr) trace_ev(p, 1 + 5 * t, s_phase - 1, __uint_as_float(s[KC - 1]));
        if (entry < 0) {
#pragma unroll
          for (int c = KH / 4; c < KC / 4; ++c) mask4(c);
        }
#pragma unroll
        for (int i = KH; i < KC; i += 4) {
          mx0 = fmaxf(mx0, __uint_as_float(s[i + 0]));
          mx1 = fmaxf(mx1, __uint_as_float(s[i + 1]));
          mx2 = fmaxf(mx2, __uint_as_float(s[i + 2]));
          mx3 = fmaxf(mx3, __uint_as_float(s[i + 3]));
        }
#else
#pragma unroll
        for (int c = 0; c < KC / 32; ++c) tmem_ld32(s_addr + c * 32, s + c * 32);
#pragma unroll
        for (int c = 0; c < KC / 32; ++c) tmem_ld_wait(s + c * 32);
        // S is in registers: the shared S buffer may take the next S.
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (k2)
            mbar_arrive_cluster(mapa_shared(smem_u32(s_free), 0));
          else
            mbar_arrive(s_free);
        }
        if (tr) trace_ev(p, 1 + 5 * t, s_phase - 1, __uint_as_float(s[KC - 1]));
        if (entry < 0) {  // partial tile: apply the position mask per element
          const int kt = entry & 0x7FFFFFFF;
          const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + kt * kTileN);
#pragma unroll
          for (int c = 0; c < KC / 4; ++c) {
            const int4 kp = __ldg(kp4 + c);
            if (kp.x > qpos) s[4 * c + 0] = __float_as_uint(-INFINITY);
            if (kp.y > qpos) s[4 * c + 1] = __float_as_uint(-INFINITY);
            if (kp.z > qpos) s[4 * c + 2] = __float_as_uint(-INFINITY);
            if (kp.w > qpos) s[4 * c + 3] = __float_as_uint(-INFINITY);
          }
        }
        float mx0 = __uint_as_float(s[0]), mx1 = __uint_as_float(s[1]);
        float mx2 = __uint_as_float(s[2]), mx3 = __uint_as_float(s[3]);
#pragma unroll
        for (int i = 4; i < KC; i += 4) {
          mx0 = fmaxf(mx0, __uint_as_float(s[i + 0]));
          mx1 = fmaxf(mx1, __uint_as_float(s[i + 1]));
          mx2 = fmaxf(mx2, __uint_as_float(s[i + 2]));
          mx3 = fmaxf(mx3, __uint_as_float(s[i + 3]));
        }
#endif
        const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
        if (tr) trace_ev(p, 2 + 5 * t, s_phase - 1, mx);
        // SoftmaxState::update (attention.cpp:209-226) with a lazy rescale:
        // the running max only moves when the tile max exceeds it by more
        // than 8 (log2 units), so P <= 2^8 and O is rescaled rarely.
        const float m_new = fmaxf(m_run, mx * sl2);
        float alpha = 1.f;
        if (m_run == -INFINITY) {
          m_run = m_new;  // first visible keys: O holds only zeros so far
        } else if (m_new > m_run + 8.f) {
          alpha = ex2(m_run - m_new);
          m_run = m_new;
        }
        const float neg = m_run == -INFINITY ? 0.f : -m_run;
        // P = exp2(S*scale*log2e - m), packed to bf16 pairs in place: word i
        // of s[] is rewritten only after s[2i], s[2i+1] were consumed.
        const float2 sc2 = make_float2(sl2, sl2), nb2 = make_float2(neg, neg);
        float2 acc2 = make_float2(0.f, 0.f);
        constexpr int kPolyPairs = HS == 64 ? USPB_FWD_POLY64 : 0;
#pragma unroll
        for (int i = 0; i < KC / 2; ++i) {
          const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, nb2);
          float2 e;
          if constexpr (kPolyPairs > 0) {
            // head size 64: the MUFU, not the tensor pipe, bounds the step
            // (2048 clk of exponentials vs 1024 of MMA per key tile), so
            // kPolyPairs of every 8 pairs go to the FMA pipe instead
            if (i % 8 < kPolyPairs) {
              e = exp2_poly2(x);
            } else {
              e.x = ex2(x.x);
              e.y = ex2(x.y);
            }
          } else {
            e.x = ex2(x.x);
            e.y = ex2(x.y);
          }
          acc2 = fadd2(acc2, e);
          // one F2FP (cvt.rn.bf16x2.f32) per pair: it does NOT share the
          // MUFU pipe on sm_100 (round 1 assumed so and packed on the integer
          // pipes, 2 IADD + PRMT per pair); measured +4 % (1294 -> 1350
          // TFLOP/s at 128K, A/B on one box, profiles/r02_fwd_ab.json)
          s[i] = pack_bf16x2(e.x, e.y);
        }
        if (tr) trace_ev(p, 3 + 5 * t, s_phase - 1, acc2.x + acc2.y);
        l_run = l_run * alpha + (acc2.x + acc2.y);
        if (j > 0) {
          // PV_t(j-1) must be done before P_t is overwritten and O_t rescaled
          if constexpr (k2)
            mbar_wait_cluster(&pv_done[t], pv_phase & 1);
          else
            mbar_wait(&pv_done[t], pv_phase & 1);
          ++pv_phase;
          tc_fence_after();
        }
#pragma unroll
        for (int c = 0; c < KC / 64; ++c) tmem_st32(p_addr + c * 32, s + c * 32);
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
          if (p.rescale_count != nullptr && lane == 0) atomicAdd(p.rescale_count, 1ull);
#pragma unroll
          for (int c = 0; c < HS / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(o_addr + c * 32, o);
            tmem_ld_wait(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(o_addr + c * 32, o);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        if constexpr (k2) {
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&p_ready[t]), 0));
        } else {
          mbar_arrive(&p_ready[t]);
        }
        if (tr) trace_ev(p, 4 + 5 * t, s_phase - 1);
      }
      const float m_use = m_run == -INFINITY ? 0.f : m_run;

      // ------------------------------------------------------------ epilogue
      if (n > 0) {  // the unit's last PV_t
        if constexpr (k2)
          mbar_wait_cluster(&pv_done[t], pv_phase & 1);
        else
          mbar_wait(&pv_done[t], pv_phase & 1);
        ++pv_phase;
        tc_fence_after();
      }
      const bool valid = q_row < p.q_len;
      const size_t row = (static_cast<size_t>(b) * p.q_len + q_row) * p.heads + h;
      const int mode = p.mode;
      const bool merge = mode == static_cast<int>(EpiMode::kMiddle) || mode == static_cast<int>(EpiMode::kLast);
      const float acc_lse = (merge && valid) ? p.lse_acc[row] : -INFINITY;  // earlier ring steps
      const float lse_t = l_run > 0.f ? m_use + log2f(l_run) : -INFINITY;  // log2 domain
      const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
      float w_run = 0.f, w_new = inv_l, lse_out = lse_t;
      if (merge) {
        const float a = acc_lse;
        const float mx = fmaxf(a, lse_t);
        if (mx == -INFINITY) {
          lse_out = -INFINITY;
          w_run = 0.f;
          w_new = 0.f;
        } else {
          lse_out = mx + log2f(exp2f(a - mx) + exp2f(lse_t - mx));
          w_run = exp2f(a - lse_out);
          w_new = exp2f(lse_t - lse_out) * inv_l;
        }
      }
      const bool write_bf16 =
          mode == static_cast<int>(EpiMode::kSingle) || mode == static_cast<int>(EpiMode::kLast);
      const bool read_acc = mode >= static_cast<int>(EpiMode::kMiddle);
      constexpr int col0 = 0;
#pragma unroll 1
      for (int c = 0; c < HS / 32; ++c) {
        float o[32];
        if (n > 0) {
          uint32_t r[32];
          tmem_ld32(o_addr + c * 32, r);
          tmem_ld_wait(r);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r[i]) * w_new;
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = 0.f;
        }
        if (!valid) continue;
        if (read_acc) {
          const float4* acc4 = reinterpret_cast<const float4*>(p.o_acc + row * HS + col0 + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 a = acc4[i];
            o[4 * i + 0] = fmaf(a.x, w_run, o[4 * i + 0]);
            o[4 * i + 1] = fmaf(a.y, w_run, o[4 * i + 1]);
            o[4 * i + 2] = fmaf(a.z, w_run, o[4 * i + 2]);
            o[4 * i + 3] = fmaf(a.w, w_run, o[4 * i + 3]);
          }
        }
        if (write_bf16) {
          uint4 w[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            w[i] = make_uint4(pack_bf16x2(o[8 * i + 0], o[8 * i + 1]), pack_bf16x2(o[8 * i + 2], o[8 * i + 3]),
                              pack_bf16x2(o[8 * i + 4], o[8 * i + 5]), pack_bf16x2(o[8 * i + 6], o[8 * i + 7]));
          uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(p.o) + (row * HS + col0 + c * 32) * 2);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = w[i];  // head-sharded O (kept for the backward)
          if (p.o_peer[0] != nullptr) {
            // direct O: the same row straight into the owning Ulysses
            // member's receive buffer (peer memory), replacing the O all-to-all
            const int part = q_row / p.o_part_rows;
            const size_t prow = static_cast<size_t>(p.o_me) * p.o_part_rows + (q_row - part * p.o_part_rows);
            uint4* rdst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(p.o_peer[part]) +
                                                   ((prow * p.heads + h) * HS + col0 + c * 32) * 2);
#pragma unroll
            for (int i = 0; i < 4; ++i) rdst[i] = w[i];
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(p.o_acc + row * HS + col0 + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(o[4 * i + 0], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        }
      }
      if (valid) {
        if (write_bf16)
          p.lse[row] = lse_out * 0.69314718055994530942f;  // natural log (attention.cpp:260)
        else
          p.lse_acc[row] = lse_out;
      }
    }
  } else {
    if constexpr (C::kRegSplit)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::kProducerRegs));
  if (warp == C::kTmaWarp) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t kv_it = 0, q_it = 0;
      const uint64_t keep = l2_policy_evict_last();
      const bool hint = p.kv_hint == 1;
      for (uint32_t it = 0;; ++it) {
        // Claim the next unit (dynamic, longest-first) and hand it to the
        // consumer roles through the ticket ring.
        const uint32_t d = it % C::kSchedDepth;
        int u;
        if (!MC || crank == 0) {
          u = atomicAdd(&p.sched[0], 1);
          mbar_wait(&sched_empty[d], ((it / C::kSchedDepth) & 1) ^ 1);
          sched_slot[d] = u;
          if constexpr (MC) {  // the same ticket to the peer CTA
            st_cluster_u32(mapa_shared(smem_u32(&sched_slot[d]), 1), static_cast<uint32_t>(u));
            mbar_arrive_cluster(mapa_shared(smem_u32(&sched_full[d]), 1));
          }
          mbar_arrive(&sched_full[d]);
        } else {  // MC peer: take the leader's ticket like a consumer
          mbar_wait_cluster(&sched_full[d], (it / C::kSchedDepth) & 1);
          u = *reinterpret_cast<const volatile int*>(&sched_slot[d]);
          mbar_arrive_cluster(mapa_shared(smem_u32(&sched_empty[d]), 0));
        }
        if (u >= p.num_units) break;
        const uint32_t unit = p.units[u];
        const int qt = unit & 0xFFFF, hp = unit_hp(unit), b = unit >> 24;
        const int beg = p.tile_off[qt];
        const int n = p.tile_off[qt + 1] - beg;
        if (n == 0) continue;
        mbar_wait(q_empty, (q_it & 1) ^ 1);
        ++q_it;
        for (int t = 0; t < NQ; ++t) {
          const int qh = p.pair_rows ? hp : hp * NQ + t;
          const int qr = (p.pair_rows ? qt * NQ + t : qt) * kTileM;
          if constexpr (k2) {  // both CTAs' Q tiles complete on the leader's barrier
            if (crank == 0) mbar_arrive_expect_tx(&q_full[t], 2 * C::kQBytes);
            const uint32_t bar = mapa_shared(smem_u32(&q_full[t]), 0);
#pragma unroll
            for (int sb = 0; sb < C::kSub; ++sb)
              tma_load_4d_2sm(sQ + t * C::kQBytes + sb * C::kSubBytes, &p.tm_q, bar, sb * 64, qh, qr, b);
          } else {
            mbar_arrive_expect_tx(&q_full[t], C::kQBytes);
#pragma unroll
            for (int sb = 0; sb < C::kSub; ++sb)
              tma_load_4d(sQ + t * C::kQBytes + sb * C::kSubBytes, &p.tm_q, &q_full[t], sb * 64, qh, qr, b);
          }
        }
        const int kvh = (p.pair_rows ? hp : hp * NQ) / group;
        for (int j = 0; j < n; ++j) {
          const int kt = p.tile_list[beg + j] & 0x7FFFFFFF;
#pragma unroll
          for (int which = 0; which < 2; ++which) {
            const uint32_t slot = kv_it % NS;
            mbar_wait(&kv_empty[slot], ((kv_it / NS) & 1) ^ 1);
            ++kv_it;
            const CUtensorMap* tm = which == 0 ? &p.tm_k : &p.tm_v;
            if constexpr (k2) {
              // my half (K: 64 key rows; V: 64 columns), completing on the leader's barrier
              if (crank == 0) mbar_arrive_expect_tx(&kv_full[slot], C::kKVBytes);
              const uint32_t bar = mapa_shared(smem_u32(&kv_full[slot]), 0);
              if (which == 0) {
#pragma unroll
                for (int sb = 0; sb < C::kSub; ++sb)
                  tma_load_4d_2sm(sKV + slot * C::kKVBytes + sb * (C::kSubBytes / 2), &p.tm_k64, bar, sb * 64, kvh,
                                  kt * kTileN + 64 * int(crank), b);
              } else {
                tma_load_4d_2sm(sKV + slot * C::kKVBytes, &p.tm_v, bar, 64 * int(crank), kvh, kt * kTileN, b);
              }
              continue;
            }
            mbar_arrive_expect_tx(&kv_full[slot], C::kKVBytes);
            if constexpr (MC) {  // my half of the tile, to both CTAs
              tma_load_4d_mc(sKV + slot * C::kKVBytes + crank * C::kSubBytes, tm, &kv_full[slot], int(crank) * 64,
                             kvh, kt * kTileN, b, uint16_t(0x3));
            } else {
#pragma unroll
              for (int sb = 0; sb < C::kSub; ++sb) {
                if (hint)
                  tma_load_4d_hint(sKV + slot * C::kKVBytes + sb * C::kSubBytes, tm, &kv_full[slot],
                                   sb * 64, kvh, kt * kTileN, b, keep);
                else
                  tma_load_4d(sKV + slot * C::kKVBytes + sb * C::kSubBytes, tm, &kv_full[slot],
                              sb * 64, kvh, kt * kTileN, b);
              }
            }
          }
        }
      }
    }
  } else if (warp == C::kMmaWarp || warp == C::kPvWarp) {
    // ------------------------------------------------------------ MMA issue
    // Two issuing warps: one serves the S = Q K^T queue, one the O += P V
    // queue. They touch disjoint TMEM (the shared S buffer vs P_t / O_t), so
    // no ordering is needed between them, and each warp's barrier waits
    // overlap the other's MMA batches (the tensor core's instruction queue
    // is shallow). Each warp runs its loop converged; one elected lane
    // issues, and its commits track only its own MMAs.
    const bool s_role = warp == C::kMmaWarp;
    {
      constexpr uint32_t kIdescQK = idesc_bf16_f32(k2 ? 256 : 128, 128, 0, 0);
      constexpr uint32_t kIdescPV = idesc_bf16_f32(k2 ? 256 : 128, HS, 0, 1);
      const uint32_t sq = smem_u32(sQ), skv = smem_u32(sKV);
      uint32_t kv_it = 0, q_phase = 0, f_phase = 0;
      uint32_t p_phase[NQ];
#pragma unroll
      for (int t = 0; t < NQ; ++t) p_phase[t] = 0;
      auto wait_full = [&](uint32_t idx) {
        if constexpr (k2)
          mbar_wait_cluster(&kv_full[idx % NS], (idx / NS) & 1);
        else
          mbar_wait(&kv_full[idx % NS], (idx / NS) & 1);
        tc_fence_after();
      };
      // commit to this CTA's barrier, or (2SM) to the same barrier of both CTAs
      auto commit = [&](uint64_t* bar) {
        if constexpr (k2) {
          if (elect_one()) mma2_commit_mc(bar, uint16_t(0x3));
          __syncwarp();
        } else {
          commit_one(bar);
        }
      };
      // Descriptor bases (16-byte units in the low bits); the batched
      // chains add the per-k-step offsets in PTX. Every MMA operand is a
      // uniform base plus a compile-time offset (TMEM base 0, stage index
      // dispatched to a constant): no per-instruction R2UR / ELECT loop.
      const uint64_t q_desc0 = smem_desc_sw128(sq, 16, 1024);
      const uint64_t kv_desc0 = smem_desc_sw128(skv, 16, 1024);
      const uint64_t v_desc0 = smem_desc_sw128(skv, C::kSubBytes, 1024);
      auto issue_qk = [&](int t, uint32_t slot) {
        dispatch_slot<NS>(slot, [&](auto S) {
          constexpr int sl = decltype(S)::value;
          const uint64_t ad = q_desc0 + static_cast<uint64_t>((t * C::kQBytes) >> 4);
          const uint64_t bd = kv_desc0 + static_cast<uint64_t>((sl * C::kKVBytes) >> 4);
          if (elect_one()) {
            if constexpr (k2)
              mma2_qk_hs128(C::kSCol, ad, bd, kIdescQK, 0u);
            else if constexpr (HS == 128)
              mma_qk_hs128(C::kSCol, ad, bd, kIdescQK, 0u);
            else
              mma_qk_hs64(C::kSCol, ad, bd, kIdescQK, 0u);
          }
          __syncwarp();
        });
      };
      auto issue_pv = [&](int t, uint32_t slot, bool acc) {
        dispatch_slot<NS>(slot, [&](auto S) {
          constexpr int sl = decltype(S)::value;
          const uint64_t bd = v_desc0 + static_cast<uint64_t>((sl * C::kKVBytes) >> 4);
          if (elect_one()) {
            if constexpr (k2)
              mma2_pv_chain(C::kOCol + t * HS, C::kPCol + t * 64, bd, kIdescPV, acc ? 1u : 0u);
            else if (acc)
              mma_pv_chain(C::kOCol + t * HS, C::kPCol + t * 64, bd, kIdescPV, 1u);
            else
              mma_pv_chain(C::kOCol + t * HS, C::kPCol + t * 64, bd, kIdescPV, 0u);
          }
          __syncwarp();
        });
      };
      uint32_t s_count = 0;  // S computations issued so far (all units)

      for (uint32_t it = 0;; ++it) {
        const int u = next_unit(sched_full, sched_empty, sched_slot, it, true);
        if (u >= p.num_units) break;
        if (k2 && crank != 0) continue;  // 2SM: the leader issues every MMA of the pair
        const int qt = p.units[u] & 0xFFFF;
        const int n = p.tile_off[qt + 1] - p.tile_off[qt];
        if (n == 0) continue;
        if (s_role) {
          // S_t(j) in (j, t) order; each needs the shared S buffer (the
          // previous S loaded into registers by its softmax) and K_j.
#pragma unroll
          for (int t = 0; t < NQ; ++t) {
            if constexpr (k2)
              mbar_wait_cluster(&q_full[t], q_phase & 1);
            else
              mbar_wait(&q_full[t], q_phase & 1);
          }
          ++q_phase;
          for (int j = 0; j < n; ++j) {
            const uint32_t ki = kv_it + 2 * j;
            wait_full(ki);
            if (lane == 0) trace_ev(p, 14, s_count / NQ);  // K_j landed (S warp)
#pragma unroll
            for (int t = 0; t < NQ; ++t) {
              if (s_count > 0) {
                if constexpr (k2)
                  mbar_wait_cluster(s_free, f_phase & 1);
                else
                  mbar_wait(s_free, f_phase & 1);
                ++f_phase;
              }
              if (t == 0 && lane == 0) trace_ev(p, 15, s_count / NQ);  // S buffer free for S_A(j)
              tc_fence_after();
              issue_qk(t, ki % NS);
              commit(&s_full[t]);
              if (lane == 0) trace_ev(p, 11 + 2 * t, j);
              ++s_count;
            }
            if constexpr (MC == 1) {
              if (elect_one()) mma_commit_mc(&kv_empty[ki % NS], uint16_t(0x3));
              __syncwarp();
            } else {
              commit(&kv_empty[ki % NS]);
            }
            if (j == n - 1) commit(q_empty);
          }
        } else {
          // PV_t(j) in (j, t) order; each needs P_t(j) and V_j.
          for (int j = 0; j < n; ++j) {
            const uint32_t vi = kv_it + 2 * j + 1;
            wait_full(vi);
#pragma unroll
            for (int t = 0; t < NQ; ++t) {
              if constexpr (k2)
                mbar_wait_cluster(&p_ready[t], p_phase[t] & 1);
              else
                mbar_wait(&p_ready[t], p_phase[t] & 1);
              if (lane == 0) trace_ev(p, 10 + 2 * t, p_phase[t]);
              ++p_phase[t];
              tc_fence_after();
              issue_pv(t, vi % NS, j > 0);
              commit(&pv_done[t]);
            }
            if constexpr (MC == 1) {
              if (elect_one()) mma_commit_mc(&kv_empty[vi % NS], uint16_t(0x3));
              __syncwarp();
            } else {
              commit(&kv_empty[vi % NS]);
            }
          }
        }
        kv_it += 2 * n;
      }
    }
  }

  }  // producer warpgroup
  if (warp == C::kTmaWarp && lane == 0 && crank == 0) {
    // The last claimer to finish resets the tickets for the next launch.
    if (atomicAdd(&p.sched[1], 1) == static_cast<int>(gridDim.x) / (MC ? 2 : 1) - 1) {
      p.sched[0] = 0;
      p.sched[1] = 0;
      __threadfence();
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync();  // no remote ticket / barrier traffic may target an exited CTA
  tc_fence_after();
  if (warp == C::kMmaWarp) {
    if constexpr (k2)
      tmem_dealloc_2sm(tmem, C::kTmemCols);
    else
      tmem_dealloc(tmem, C::kTmemCols);
  }
}

// --------------------------------------------------------------- launchers
template <int NQ, int HS, int MC = 0>
static cudaError_t launch_impl(const FwdParams& p, int grid, cudaStream_t stream) {
  using C = FwdCfg<NQ, HS>;
  auto kern = fa_fwd_sm100_kernel<NQ, HS, MC>;
  static std::atomic<uint64_t> attr_done{0};  // per instantiation and device
  const cudaError_t e = ensure_smem_attr(kern, C::kSmemBytes, attr_done);
  if (e != cudaSuccess) return e;
  if constexpr (MC > 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid & ~1), 1, 1);
    cfg.blockDim = dim3(C::kThreads, 1, 1);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
  }
  kern<<<grid, C::kThreads, C::kSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fa_fwd(const FwdParams& p, int nq, int hs, int grid, cudaStream_t stream) {
  if (p.cluster) {
    if (nq != 2 || hs != 128 || p.pair_rows) return cudaErrorInvalidValue;
#ifdef USPB_DEV_2SM
    // development build only: cta_group::2 MMAs (measured 886 vs 1276
    // TFLOP/s for the multicast clusters)
    if (p.cluster == 2) return launch_impl<2, 128, 2>(p, grid, stream);
#else
    if (p.cluster == 2) return cudaErrorNotSupported;
#endif
    return launch_impl<2, 128, 1>(p, grid, stream);
  }
  if (nq == 2 && hs == 128) return launch_impl<2, 128>(p, grid, stream);
  if (nq == 1 && hs == 128) return launch_impl<1, 128>(p, grid, stream);
  if (nq == 2 && hs == 64) return launch_impl<2, 64>(p, grid, stream);
  if (nq == 1 && hs == 64) return launch_impl<1, 64>(p, grid, stream);
  return cudaErrorInvalidValue;
}

}  // namespace uspb200
