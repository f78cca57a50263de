// fa_bwd_sm100.cu — attention backward for sm_100a.
//
// Restates attention_block_backward (reference src/numerics/attention.cpp:
// 282-324) and output_dot_rows (:266-280) with tcgen05 MMAs:
//
//   dq kernel   (unit = batch, q head, 128-row q tile; loop over key tiles)
//       S = Q K^T, dP = dO V^T            (SS MMAs into TMEM)
//       dS = P (dP - delta), P = exp(S/sqrt(hs) - lse)   (4 compute warps)
//       dQ += dS K                         (TS MMA, dS bf16 over S in TMEM)
//   dkdv kernel (unit = batch, kv head, 128-row key tile; loop over the GQA
//                group's q heads x q tiles)
//       S^T = K Q^T, dP^T = V dO^T
//       P^T, dS^T as above (thread = key row)
//       dV += P^T dO,  dK += dS^T Q        (TS MMAs)
//
// Same machinery as the forward (fa_fwd_sm100.cu): TMA-fed 128B-swizzled
// tiles, one elected thread issuing batched MMA chains, mbarrier pipelines,
// dynamic unit tickets. Results accumulate in fp32 (ring steps add into
// them); the host casts to bf16 at the end.
#include <cuda_runtime.h>
#include <math.h>

#include <type_traits>

#include "fa_bwd.hpp"
#include "fa_fwd.hpp"
#include "ptx_sm100.cuh"

#ifndef USPB_DQ_KSLOTS
#define USPB_DQ_KSLOTS 3
#endif
#ifndef USPB_DBG_NOEXP
#define USPB_DBG_NOEXP 0
#endif
#ifndef USPB_DBG_NOCOMPUTE
#define USPB_DBG_NOCOMPUTE 0
#endif
#ifndef USPB_DKDV_PAIRW
#define USPB_DKDV_PAIRW 1  // one hand-off barrier per chunk pair (see the dK/dV kernel)
#endif
#ifndef USPB_DKDV_QD1
#define USPB_DKDV_QD1 0  // 1: Q and dO of a q tile on one barrier (measured slower, 247 -> 255 ms: S(i+1) then waits for dO)
#endif
#ifndef USPB_DKDV_SWAP
#define USPB_DKDV_SWAP 1  // Q / dO slot roles alternate per ring round (qd_slot)
#endif
#ifndef USPB_FUSED_RDEPTH
#define USPB_FUSED_RDEPTH 1
#endif
#ifndef USPB_FUSED_DYN
#define USPB_FUSED_DYN 1  // the fused kernel's MMA warp issues S^T(g+1) / dQ(g)+dK(g) in readiness order
#endif
#ifndef USPB_FUSED_NORED
#define USPB_FUSED_NORED 0  // development A/B: the fused kernel's drain skips the dQ reductions
#endif
#ifndef USPB_DKDV_STAGES
#define USPB_DKDV_STAGES 6
#endif

namespace uspb200 {
namespace {

using namespace ptx;

template <int N, class F>
__device__ __forceinline__ void bwd_dispatch_slot(uint32_t slot, F&& f) {
  if constexpr (N > 0) {
    if (slot == N - 1)
      f(std::integral_constant<int, N - 1>{});
    else
      bwd_dispatch_slot<N - 1>(slot, f);
  }
}

__device__ __forceinline__ void bwd_trace(const BwdParams& p, int ev, uint32_t i) {
#ifdef USPB_TRACE
  if (p.trace != nullptr && blockIdx.x == 0 && i < static_cast<uint32_t>(kTraceTiles)) {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    p.trace[ev * kTraceTiles + i] = c;
  }
#else
  (void)p, (void)ev, (void)i;
#endif
}

__device__ __forceinline__ void bwd_commit(uint64_t* bar) {
  if (elect_one()) mma_commit(bar);
  __syncwarp();
}

#ifndef USPB_BWD_F2FP
#define USPB_BWD_F2FP 1  // F2FP packing: +3 % (839 -> 865 TFLOP/s at 128K, A/B)
#endif
// bf16x2 packing of P / dS: F2FP (cvt.rn) or the integer-pipe round-half-up
__device__ __forceinline__ uint32_t bwd_pack(float lo, float hi) {
  return USPB_BWD_F2FP ? pack_bf16x2(lo, hi) : pack_bf16x2_int(lo, hi);
}

template <int HS>
struct BwdCfg {
  static constexpr int kTile = 128;
  static constexpr int kTileBytes = kTile * HS * 2;  // one 128-row bf16 tile
  static constexpr int kSubBytes = 128 * 128;
  static constexpr int kSub = HS / 64;
  // 8 compute warps (two per TMEM lane quarter, each owning half of the
  // tile's columns), the TMA warp and the MMA warp
  static constexpr int kCompute = 8;
  // three full warpgroups (warps 10, 11 idle) so setmaxnreg can move
  // registers to the compute warps: per SM sub-partition 2 x 208 + 1 x 88
  // (384 threads x 168 at launch); without it 10 warps cap every thread at
  // 168 registers and the compute warps spill
  static constexpr int kThreads = 32 * (kCompute + 4);
  static constexpr int kComputeRegs = 208, kProducerRegs = 88;
  static_assert(kCompute * 32 * kComputeRegs + 128 * kProducerRegs <= kThreads * 168, "register split");
  static constexpr int kTmaWarp = kCompute, kMmaWarp = kCompute + 1;
  static constexpr int kBudget = 227 * 1024 - 4096;
  static constexpr int kStages = (kBudget - 2 * kTileBytes) / kTileBytes > USPB_DKDV_STAGES
                                     ? USPB_DKDV_STAGES
                                     : (kBudget - 2 * kTileBytes) / kTileBytes;
  static constexpr int kVecBytes = 3 * 128 * 4;  // -lse2 | -delta | q position of one q tile
  static constexpr int kSmemBytes = 1024 + 2 * kTileBytes + kStages * kTileBytes + 2048 + kStages * kVecBytes;
  // dq kernel: K tiles in a 3-slot ring (released after the tile's dQ MMAs),
  // V tiles in a 2-slot ring (released as soon as dP has been computed)
  static constexpr int kKSlots = USPB_DQ_KSLOTS, kVSlots = 2;
  static constexpr int kDqSmemBytes = 1024 + (2 + kKSlots + kVSlots) * kTileBytes + 512;
  static_assert(kDqSmemBytes <= 227 * 1024, "dq smem");
  static constexpr uint32_t kIdescSS = idesc_bf16_f32(128, 128, 0, 0);  // S / dP
  static constexpr uint32_t kIdescTS = idesc_bf16_f32(128, HS, 0, 1);   // acc += X * tile
  static_assert(kStages >= 2 && kStages % 2 == 0, "smem; Q / dO slot pairs");
};

// The 32-column chunks of a tile in the order their packed operands become
// ready (warp half 0 does chunks 0,1, half 1 does 2,3, concurrently).
// dK/dV Q / dO ring: position 2T + w (w = 0 Q, 1 dO of the T-th q tile of
// this CTA) -> slot. Tile T uses the slot pair 2 (T mod NS/2); with SWAP the
// roles alternate per round, so Q(T + NS/2) lands in dO(T)'s slot, which is
// released right after the dV(T) MMAs — one phase before Q(T)'s slot (after
// dK(T)) — and the next S^T's operand arrives earlier.
template <int NS>
__device__ __forceinline__ uint32_t qd_slot(uint32_t pos) {
  const uint32_t t = pos >> 1, w = pos & 1u, round = t / (NS / 2);
  return 2u * (t % (NS / 2)) + (w ^ (USPB_DKDV_SWAP ? (round & 1u) : 0u));
}
__device__ __forceinline__ int chunk_at(int n) { return ((n & 1) << 1) | (n >> 1); }
// TMEM column (within an S / dP buffer) of chunk c's packed bf16 result:
// each warp half writes only inside the 64 columns it reads (half 0 owns
// [0,64), half 1 [64,128)), after it has consumed them, so the two halves
// never race.
__device__ __forceinline__ uint32_t packed_col(int c) { return static_cast<uint32_t>((c >> 1) * 64 + (c & 1) * 16); }

__device__ __forceinline__ void st16(uint32_t addr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// Epilogue helper: rows of one 128-row tile, `cols` fp32 columns from TMEM
// starting at `col`, scaled, (accumulated into) dst row-major.
template <int NCOL>
__device__ __forceinline__ void store_rows(uint32_t lane_base, uint32_t col, bool have, bool valid, float* dst,
                                           float sc, bool accumulate) {
#pragma unroll 1
  for (int c = 0; c < NCOL / 32; ++c) {
    uint32_t r[32];
    if (have) {
      tmem_ld32(lane_base + col + c * 32, r);
      tmem_ld_wait(r);
    }
    if (!valid) continue;
    float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 v = have ? make_float4(__uint_as_float(r[4 * i]) * sc, __uint_as_float(r[4 * i + 1]) * sc,
                                    __uint_as_float(r[4 * i + 2]) * sc, __uint_as_float(r[4 * i + 3]) * sc)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      if (accumulate) {
        const float4 a = d4[i];
        v.x += a.x;
        v.y += a.y;
        v.z += a.z;
        v.w += a.w;
      }
      d4[i] = v;
    }
  }
}

// ============================================================ dq kernel
// TMEM: S0 [0,128), dP [128,256), dQ [256,256+HS), S1 [384,512) (HS = 128;
// for HS = 64 the same columns). dS (bf16) is written over consumed columns
// of the S buffer it came from (packed_col). S(j+1) goes to the other S buffer
// while tile j's elementwise work runs; dQ k-steps are issued per 32-key
// chunk as soon as that chunk's dS is in TMEM.
// MC = 1: a 2-CTA cluster runs the two q heads of a head pair (same kv
// head) over the same q tile; each CTA loads one 64-column half of every
// K / V tile and multicasts it to both (unit hp field = head pair).
template <int HS, int MC>
__global__ void __launch_bounds__(BwdCfg<HS>::kThreads, 1) fa_bwd_dq_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdCfg<HS>;
  static_assert(!MC || HS == 128, "cluster mode needs two 64-column halves");
  constexpr int NK = C::kKSlots, NV = C::kVSlots;
  constexpr uint32_t kDP = 128, kDQ = 256, kS1 = 384;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sDO = smem + C::kTileBytes;
  uint8_t* sK = smem + 2 * C::kTileBytes;   // [NK]
  uint8_t* sV = sK + NK * C::kTileBytes;     // [NV]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + NV * C::kTileBytes);
  uint64_t* q_full = bars;            // Q + dO landed
  uint64_t* q_empty = bars + 1;
  uint64_t* s_full = bars + 2;        // [2] S buffer b computed
  uint64_t* dp_full = bars + 4;       // dP computed
  // [2][4] dS chunk in TMEM (128 arrivals), by tile parity: the compute
  // warps may finish tile j+1's chunks before the MMA warp has waited for
  // tile j's (dP(j+1) is issued ahead of tile j's dQ MMAs)
  uint64_t* chunk_ready = bars + 5;
  uint64_t* dq_full = bars + 13;      // unit's last dQ MMA done
  uint64_t* k_full = bars + 14;       // [NK]
  uint64_t* k_empty = k_full + NK;    // [NK]
  uint64_t* v_full = k_empty + NK;    // [NV]
  uint64_t* v_empty = v_full + NV;    // [NV]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + NV);
  int* unit_slot = reinterpret_cast<int*>(tmem_slot + 2);
  uint64_t* u_full = reinterpret_cast<uint64_t*>(unit_slot + 2);
  uint64_t* u_empty = u_full + 1;
  uint64_t* dp_free = u_empty + 1;    // tile's dP loaded by every compute warp

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(dp_free, C::kCompute);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(dp_full, 1);
    // with PAIRW, barrier (parity, k) collects chunk k of both warp halves
    for (int c = 0; c < 8; ++c) mbar_init(&chunk_ready[c], USPB_DKDV_PAIRW ? 256 : 128);
    mbar_init(dq_full, 1);
    mbar_init(u_full, 1);
    // compute warps + MMA warp (of both CTAs, + the peer's TMA warp, with MC)
    mbar_init(u_empty, MC ? 2 * (C::kCompute + 1) + 1 : C::kCompute + 1);
    for (int s = 0; s < NK; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], MC ? 2 : 1);
    }
    for (int s = 0; s < NV; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], MC ? 2 : 1);
    }
    fence_barrier_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync();  // the peer's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t crank = MC ? cluster_ctarank() : 0u;
  auto unit_head = [&](uint32_t unit) {
    return MC ? int((unit >> 16) & 0xFF) * 2 + int(crank) : int((unit >> 16) & 0xFF);
  };
  const uint32_t tmem = *tmem_slot;
  if (tmem != 0) __trap();
  const int group = p.heads / p.kv_heads;

  auto get_unit = [&](uint32_t it) {
    if constexpr (MC)
      mbar_wait_cluster(u_full, it & 1);
    else
      mbar_wait(u_full, it & 1);
    const int u = *reinterpret_cast<volatile int*>(unit_slot);
    __syncwarp();
    if (lane == 0) {
      if constexpr (MC)
        mbar_arrive_cluster(mapa_shared(smem_u32(u_empty), 0));  // the leader's slot
      else
        mbar_arrive(u_empty);
    }
    return u;
  };

  if (warp >= C::kCompute) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::kProducerRegs));
  if (warp < C::kCompute) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::kComputeRegs));
    // ---------------------------------------------------- compute warps
    const int q4 = warp & 3, hf = warp >> 2;
    const int row_in_tile = q4 * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const float sl2 = p.scale_log2;
    uint32_t g = 0, d_phase = 0;  // g: running tile counter (buffer parity, phases)
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it);
      if (u >= p.num_units) break;
      const uint32_t unit = p.units[u];
      const int qt = unit & 0xFFFF, h = unit_head(unit), b = unit >> 24;
      const int beg = p.tile_off[qt], n = p.tile_off[qt + 1] - beg;
      const int q_row = qt * 128 + row_in_tile;
      const bool valid = q_row < p.q_len;
      const size_t row = (static_cast<size_t>(b) * p.q_len + (valid ? q_row : 0)) * p.heads + h;
      const float lse2 = valid ? p.lse[row] * 1.4426950408889634f : 0.f;
      const float dlt = valid ? p.delta[row] : 0.f;
      const int qpos = p.q_pos[q_row];
      for (int j = 0; j < n; ++j, ++g) {
        const int entry = p.tile_list[beg + j];
        const uint32_t sb = (g & 1) ? kS1 : 0u;
        const bool tr = q4 == 0 && lane == 0;
        mbar_wait(&s_full[g & 1], (g >> 1) & 1);
        if (tr) bwd_trace(p, 4 * hf + 0, g);
        mbar_wait(dp_full, g & 1);
        if (tr) bwd_trace(p, 4 * hf + 1, g);
        tc_fence_after();
        // Both of this warp's chunks of S and dP into registers at once, so
        // the dP buffer is released before the elementwise work: dP(j+1) is
        // computed while this tile's dS is formed.
        uint32_t s2[64], dp2[64];
        tmem_ld32(lane_base + sb + (2 * hf) * 32, s2);
        tmem_ld32(lane_base + sb + (2 * hf + 1) * 32, s2 + 32);
        tmem_ld32(lane_base + kDP + (2 * hf) * 32, dp2);
        tmem_ld32(lane_base + kDP + (2 * hf + 1) * 32, dp2 + 32);
        tmem_ld_wait(s2);
        tmem_ld_wait(dp2);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dp_free);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c = 2 * hf + cc;
          uint32_t* s = s2 + 32 * cc;
          const uint32_t* dp = dp2 + 32 * cc;
          if (entry < 0) {
            const int kt = entry & 0x7FFFFFFF;
            const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + kt * 128 + c * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int4 kp = __ldg(kp4 + i);
              if (kp.x > qpos) s[4 * i + 0] = __float_as_uint(-INFINITY);
              if (kp.y > qpos) s[4 * i + 1] = __float_as_uint(-INFINITY);
              if (kp.z > qpos) s[4 * i + 2] = __float_as_uint(-INFINITY);
              if (kp.w > qpos) s[4 * i + 3] = __float_as_uint(-INFINITY);
            }
          }
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {  // packed fp32x2: one issue slot per pair
            const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])),
                                   make_float2(sl2, sl2), make_float2(-lse2, -lse2));
            const float2 pr = make_float2(ex2(x.x), ex2(x.y));
            const float2 d = fadd2(make_float2(__uint_as_float(dp[2 * i]), __uint_as_float(dp[2 * i + 1])),
                                   make_float2(-dlt, -dlt));
            const float2 ds = fmul2(pr, d);
            pk[i] = bwd_pack(ds.x, ds.y);
          }
          st16(lane_base + sb + packed_col(c), pk);  // dS chunk c, over already-consumed S columns
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&chunk_ready[(g & 1) * 4 + (USPB_DKDV_PAIRW ? cc : c)]);
        }
        if (tr) bwd_trace(p, 4 * hf + 2, g);
      }
      // epilogue: dq (+)= dQ / sqrt(hs); warp half hf stores half the columns
      if (n > 0) {
        mbar_wait(dq_full, d_phase & 1);
        ++d_phase;
        tc_fence_after();
      }
      store_rows<HS / 2>(lane_base, kDQ + hf * (HS / 2), n > 0, valid, p.dq + row * HS + hf * (HS / 2),
                         p.inv_scale, p.accumulate != 0);
    }
  } else if (warp == C::kTmaWarp) {
    // ---------------------------------------------------- producer
    if (lane == 0) {
      uint32_t kv_it = 0, q_it = 0;
      for (uint32_t it = 0;; ++it) {
        int u;
        if (!MC || crank == 0) {
          u = atomicAdd(&p.sched[0], 1);
          mbar_wait(u_empty, (it & 1) ^ 1);
          *reinterpret_cast<volatile int*>(unit_slot) = u;
          if constexpr (MC) {  // the same ticket to the peer CTA
            st_cluster_u32(mapa_shared(smem_u32(unit_slot), 1), static_cast<uint32_t>(u));
            mbar_arrive_cluster(mapa_shared(smem_u32(u_full), 1));
          }
          mbar_arrive(u_full);
        } else {  // MC peer: take the leader's ticket
          mbar_wait_cluster(u_full, it & 1);
          u = *reinterpret_cast<volatile int*>(unit_slot);
          mbar_arrive_cluster(mapa_shared(smem_u32(u_empty), 0));
        }
        if (u >= p.num_units) break;
        const uint32_t unit = p.units[u];
        const int qt = unit & 0xFFFF, h = unit_head(unit), b = unit >> 24;
        const int beg = p.tile_off[qt], n = p.tile_off[qt + 1] - beg;
        if (n == 0) continue;
        mbar_wait(q_empty, (q_it & 1) ^ 1);
        ++q_it;
        mbar_arrive_expect_tx(q_full, 2 * C::kTileBytes);
        for (int sb = 0; sb < C::kSub; ++sb) {
          tma_load_4d(sQ + sb * C::kSubBytes, &p.tm_q, q_full, sb * 64, h, qt * 128, b);
          tma_load_4d(sDO + sb * C::kSubBytes, &p.tm_do, q_full, sb * 64, h, qt * 128, b);
        }
        const int kvh = h / group;
        for (int j = 0; j < n; ++j, ++kv_it) {
          const int kt = p.tile_list[beg + j] & 0x7FFFFFFF;
          const uint32_t ks = kv_it % NK, vs = kv_it % NV;
          mbar_wait(&k_empty[ks], ((kv_it / NK) & 1) ^ 1);
          bwd_trace(p, 14, kv_it);
          mbar_arrive_expect_tx(&k_full[ks], C::kTileBytes);
          if constexpr (MC) {  // my half of the tile, to both CTAs
            tma_load_4d_mc(sK + ks * C::kTileBytes + crank * C::kSubBytes, &p.tm_k, &k_full[ks], int(crank) * 64,
                           kvh, kt * 128, b, uint16_t(0x3));
          } else {
            for (int sb = 0; sb < C::kSub; ++sb)
              tma_load_4d(sK + ks * C::kTileBytes + sb * C::kSubBytes, &p.tm_k, &k_full[ks], sb * 64, kvh,
                          kt * 128, b);
          }
          mbar_wait(&v_empty[vs], ((kv_it / NV) & 1) ^ 1);
          bwd_trace(p, 15, kv_it);
          mbar_arrive_expect_tx(&v_full[vs], C::kTileBytes);
          if constexpr (MC) {
            tma_load_4d_mc(sV + vs * C::kTileBytes + crank * C::kSubBytes, &p.tm_v, &v_full[vs], int(crank) * 64,
                           kvh, kt * 128, b, uint16_t(0x3));
          } else {
            for (int sb = 0; sb < C::kSub; ++sb)
              tma_load_4d(sV + vs * C::kTileBytes + sb * C::kSubBytes, &p.tm_v, &v_full[vs], sb * 64, kvh,
                          kt * 128, b);
          }
        }
      }
      if (crank == 0 && atomicAdd(&p.sched[1], 1) == static_cast<int>(gridDim.x) / (MC ? 2 : 1) - 1) {
        p.sched[0] = 0;
        p.sched[1] = 0;
        __threadfence();
      }
    }
  } else if (warp == C::kMmaWarp) {
    // ---------------------------------------------------- MMA issue
    const uint64_t q_desc = smem_desc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t do_desc = smem_desc_sw128(smem_u32(sDO), 16, 1024);
    const uint64_t k_desc0 = smem_desc_sw128(smem_u32(sK), 16, 1024);
    const uint64_t v_desc0 = smem_desc_sw128(smem_u32(sV), 16, 1024);
    const uint64_t kmn_desc0 = smem_desc_sw128(smem_u32(sK), C::kSubBytes, 1024);
    uint32_t kv_it = 0, q_phase = 0, g = 0;
    // D = A * B^T with B K-major: a K tile (S) or a V tile (dP) from its ring
    auto ss = [&](uint32_t d, uint64_t ad, uint64_t b0, uint32_t slot, auto nslots) {
      bwd_dispatch_slot<decltype(nslots)::value>(slot, [&](auto S) {
        constexpr int sl = decltype(S)::value;
        const uint64_t bd = b0 + static_cast<uint64_t>((sl * C::kTileBytes) >> 4);
        if (elect_one()) {
          if constexpr (HS == 128)
            mma_qk_hs128(d, ad, bd, C::kIdescSS, 0u);
          else
            mma_qk_hs64(d, ad, bd, C::kIdescSS, 0u);
        }
        __syncwarp();
      });
    };
    using KN = std::integral_constant<int, NK>;
    using VN = std::integral_constant<int, NV>;
    auto issue_s = [&](uint32_t t, uint32_t buf) {  // S(t) = Q K(t)^T
      mbar_wait(&k_full[t % NK], (t / NK) & 1);
      tc_fence_after();
      ss(buf, q_desc, k_desc0, t % NK, KN{});
    };
    auto issue_dp = [&](uint32_t t) {  // dP(t) = dO V(t)^T; V(t) is free afterwards
      mbar_wait(&v_full[t % NV], (t / NV) & 1);
      tc_fence_after();
      ss(kDP, do_desc, v_desc0, t % NV, VN{});
      bwd_commit(dp_full);
      if constexpr (MC) {  // V(t) is free in both CTAs once both MMA warps used it
        if (elect_one()) mma_commit_mc(&v_empty[t % NV], uint16_t(0x3));
        __syncwarp();
      } else {
        bwd_commit(&v_empty[t % NV]);
      }
    };
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it);
      if (u >= p.num_units) break;
      const int qt = p.units[u] & 0xFFFF;
      const int n = p.tile_off[qt + 1] - p.tile_off[qt];
      if (n == 0) continue;
      mbar_wait(q_full, q_phase & 1);
      ++q_phase;
      issue_s(kv_it, (g & 1) ? kS1 : 0u);  // S(0)
      bwd_commit(&s_full[g & 1]);
      if (g > 0) mbar_wait(dp_free, (g - 1) & 1);  // the previous tile's dP was loaded
      issue_dp(kv_it);                              // dP(0)
      for (int j = 0; j < n; ++j, ++g) {
        const uint32_t t = kv_it + j;
        if (j + 1 < n) {
          // S(j+1) into the other buffer and dP(j+1) as soon as tile j's dP
          // is in registers: both overlap tile j's elementwise work
          issue_s(t + 1, ((g + 1) & 1) ? kS1 : 0u);
          bwd_commit(&s_full[(g + 1) & 1]);
          if (lane == 0) bwd_trace(p, 8, g);
          mbar_wait(dp_free, g & 1);
          if (lane == 0) bwd_trace(p, 9, g);
          issue_dp(t + 1);
          if (lane == 0) bwd_trace(p, 10, g);
        } else {
          bwd_commit(q_empty);  // every MMA reading Q / dO has been issued
        }
        const uint32_t sb = (g & 1) ? kS1 : 0u;
        // dQ += dS K, chunk by chunk (K tile as the MN-major B operand)
        bwd_dispatch_slot<NK>(t % NK, [&](auto S) {
          constexpr int sl = decltype(S)::value;
          const uint64_t bd = kmn_desc0 + static_cast<uint64_t>((sl * C::kTileBytes) >> 4);
#pragma unroll
          for (int n4 = 0; n4 < 4; ++n4) {
            const int c = chunk_at(n4);
            if (!USPB_DKDV_PAIRW || (n4 & 1) == 0) {
              mbar_wait(&chunk_ready[(g & 1) * 4 + (USPB_DKDV_PAIRW ? n4 >> 1 : c)], (g >> 1) & 1);
              if (lane == 0) bwd_trace(p, 11 + (n4 >> 1), g);
              tc_fence_after();
            }
            if (elect_one())
              mma_ts_k2(kDQ, sb + packed_col(c), bd + static_cast<uint64_t>(c * 256), C::kIdescTS,
                        (j > 0 || n4 > 0) ? 1u : 0u);
            __syncwarp();
          }
        });
        if constexpr (MC) {
          if (elect_one()) mma_commit_mc(&k_empty[t % NK], uint16_t(0x3));
          __syncwarp();
        } else {
          bwd_commit(&k_empty[t % NK]);
        }
      }
      bwd_commit(dq_full);
      kv_it += n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync();  // no remote traffic may target an exited CTA
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, 512);
}

// ============================================================ dk/dv kernel
// TMEM: S^T [0,128) (P^T bf16 over consumed columns), dP^T [128,256)
// (dS^T bf16 likewise), dV [256, 256+HS), dK [256+HS, 256+2HS).
// Q / dO tiles stream through the slot ring; K, V stay resident per unit.
// dV / dK k-steps are issued per 32-query chunk as soon as that chunk's
// P^T / dS^T are in TMEM.
// MC = 1: a 2-CTA cluster runs the two key tiles of a key-tile pair (units
// and CSR over pairs, transpose_plan_pairs): both walk the same q-tile list
// (the union of the two tiles'), each CTA TMA-loads one 64-column half of
// every Q / dO tile multicast to both, and a slot is refilled once both MMA
// warps released it (count-2 empty barriers, multicast commits). Halves the
// L2 -> SM traffic of the streamed operands; K / V stay per CTA.
template <int HS, int MC>
__global__ void __launch_bounds__(BwdCfg<HS>::kThreads, 1) fa_bwd_dkdv_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdCfg<HS>;
  static_assert(!MC || HS == 128, "cluster mode needs two 64-column halves");
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + C::kTileBytes;
  uint8_t* sQD = smem + 2 * C::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sQD + NS * C::kTileBytes);
  uint64_t* kv_full = bars;          // K + V landed
  uint64_t* kv_empty = bars + 1;
  uint64_t* s_full = bars + 2;       // S^T in TMEM
  uint64_t* p_ready = bars + 3;      // [4] P^T chunk written (128 arrivals)
  uint64_t* acc_full = bars + 7;     // unit's last dV/dK MMA done
  uint64_t* dp_full = bars + 8;      // dP^T in TMEM
  uint64_t* ds_ready = bars + 9;     // [4] dS^T chunk written (128 arrivals)
  uint64_t* qd_full = bars + 13;     // [NS]
  uint64_t* qd_empty = qd_full + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qd_empty + NS);
  int* unit_slot = reinterpret_cast<int*>(tmem_slot + 2);
  uint64_t* u_full = reinterpret_cast<uint64_t*>(unit_slot + 2);
  uint64_t* u_empty = u_full + 1;
  // [NS slots][-lse2 128 | -delta 128 | qpos 128]: the vector of the q tile whose
  // Q sits in ring slot s, bulk-copied by the TMA warp with that Q tile
  uint8_t* vec = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(u_empty + 1) + 15u) & ~uintptr_t(15));
  const uint32_t vec_s = smem_u32(vec);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    for (int c = 0; c < 4; ++c) {
      // PAIRW: barrier k collects chunk k of both warp halves (chunks k and
      // 2 + k land together), so the MMA warp waits twice per phase, not 4x
      mbar_init(&p_ready[c], USPB_DKDV_PAIRW ? 256 : 128);
      mbar_init(&ds_ready[c], USPB_DKDV_PAIRW ? 256 : 128);
    }
    mbar_init(acc_full, 1);
    mbar_init(u_full, 1);
    // compute warps + MMA warp (of both CTAs, + the peer's TMA warp, with MC)
    mbar_init(u_empty, MC ? 2 * (C::kCompute + 1) + 1 : C::kCompute + 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&qd_full[s], 1);
      mbar_init(&qd_empty[s], MC ? 2 : 1);
    }
    fence_barrier_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync();  // the peer's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t crank = MC ? cluster_ctarank() : 0u;
  // CSR row of a unit (key tile, or key-tile pair with MC) and this CTA's key tile
  auto unit_row = [](uint32_t unit) { return int(unit & 0xFFFF); };
  auto unit_ktile = [&](uint32_t unit) { return MC ? int(unit & 0xFFFF) * 2 + int(crank) : int(unit & 0xFFFF); };
  const uint32_t tmem = *tmem_slot;
  if (tmem != 0) __trap();
  const int group = p.heads / p.kv_heads;

  auto get_unit = [&](uint32_t it) {
    if constexpr (MC)
      mbar_wait_cluster(u_full, it & 1);
    else
      mbar_wait(u_full, it & 1);
    const int u = *reinterpret_cast<volatile int*>(unit_slot);
    __syncwarp();
    if (lane == 0) {
      if constexpr (MC)
        mbar_arrive_cluster(mapa_shared(smem_u32(u_empty), 0));  // the leader's slot
      else
        mbar_arrive(u_empty);
    }
    return u;
  };

  if (warp >= C::kCompute) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::kProducerRegs));
  if (warp < C::kCompute) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::kComputeRegs));
    // ---------------------------------------------------- compute warps (thread = key row)
    const int q4 = warp & 3, hf = warp >> 2;
    const int key_in_tile = q4 * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const float sl2 = p.scale_log2;
    uint32_t g = 0, a_phase = 0;
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it);
      if (u >= p.num_units) break;
      const uint32_t unit = p.units[u];
      const int kt = unit_ktile(unit), row = unit_row(unit), kvh = (unit >> 16) & 0xFF, b = unit >> 24;
      const int beg = p.tile_off[row], n = p.tile_off[row + 1] - beg;
      const int k_row = kt * 128 + key_in_tile;
      const int kpos = p.k_pos[k_row];
      // Per q tile, lse2 / delta / q positions of its 128 rows go through
      // shared memory (a parity-double-buffered 3 x 128 vector). Their global
      // loads are issued one q tile ahead, so the L2 latency hides behind
      // the previous tile's MMAs and elementwise work.
      const int total = group * n;
      for (int i = 0; i < total; ++i, ++g) {
        const int entry = p.tile_list[beg + i % n];
        // this q tile's lse2 / delta / positions came with its Q tile (ring
        // slot qd_slot(2g); the slot is not refilled before this tile's dK MMAs)
        const uint32_t qslot = qd_slot<NS>(2 * g);
        mbar_wait(&qd_full[qslot], ((2 * g) / NS) & 1);
        const uint32_t vb = vec_s + qslot * C::kVecBytes;
        // phase 1: P^T = exp(S^T - lse) (thread = key row), packed over the
        // consumed S^T columns for the dV MMAs; fp32 P kept for phase 2
        const bool tr = q4 == 0 && lane == 0;
        mbar_wait(s_full, g & 1);
        if (tr) bwd_trace(p, 4 * hf + 0, g);
        tc_fence_after();
        uint32_t pp2[2][16];  // bf16 P^T pairs, reused by phase 2
        // both 32-column chunks of this warp in flight at once (one TMEM
        // round trip per phase instead of two)
        uint32_t sv2[64];
        tmem_ld32(lane_base + (2 * hf) * 32, sv2);
        tmem_ld32(lane_base + (2 * hf + 1) * 32, sv2 + 32);
        tmem_ld_wait(sv2);
        tmem_ld_wait(sv2 + 32);
        // the mask test is hoisted out of the element loop: one straight-line
        // block per chunk for the (common) full tiles
        auto p_chunks = [&](auto masked) {
          constexpr bool kMasked = decltype(masked)::value;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = 2 * hf + cc;
            const uint32_t* sv = sv2 + 32 * cc;
            uint32_t* pp = pp2[cc];
#pragma unroll
            for (int i4 = 0; i4 < (USPB_DBG_NOCOMPUTE ? 0 : 8); ++i4) {
              const uint32_t col = (c * 32 + 4 * i4) * 4;
              const float4 L4 = lds_f4(vb + col);  // -lse2 of 4 q rows
              const float2 x01 = ffma2(make_float2(__uint_as_float(sv[4 * i4]), __uint_as_float(sv[4 * i4 + 1])),
                                       make_float2(sl2, sl2), make_float2(L4.x, L4.y));
              const float2 x23 = ffma2(make_float2(__uint_as_float(sv[4 * i4 + 2]), __uint_as_float(sv[4 * i4 + 3])),
                                       make_float2(sl2, sl2), make_float2(L4.z, L4.w));
#if USPB_DBG_NOEXP
              float pv[4] = {x01.x, x01.y, x23.x, x23.y};
#else
              float pv[4] = {ex2(x01.x), ex2(x01.y), ex2(x23.x), ex2(x23.y)};
#endif
              if constexpr (kMasked) {
                const float4 Q4 = lds_f4(vb + 1024 + col);
                const int qv[4] = {__float_as_int(Q4.x), __float_as_int(Q4.y), __float_as_int(Q4.z),
                                   __float_as_int(Q4.w)};
#pragma unroll
                for (int e = 0; e < 4; ++e) pv[e] = kpos > qv[e] ? 0.f : pv[e];
              }
              pp[2 * i4] = bwd_pack(pv[0], pv[1]);
              pp[2 * i4 + 1] = bwd_pack(pv[2], pv[3]);
            }
            st16(lane_base + packed_col(c), pp);
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_ready[USPB_DKDV_PAIRW ? cc : c]);
          }
        };
        if (entry < 0)
          p_chunks(std::true_type{});
        else
          p_chunks(std::false_type{});
        if (tr) bwd_trace(p, 4 * hf + 1, g);
        // phase 2: dS^T = P^T (dP^T - delta), packed over the consumed dP^T
        // columns for the dK MMAs (S^T(i+1) is computed meanwhile)
        mbar_wait(dp_full, g & 1);
        if (tr) bwd_trace(p, 4 * hf + 2, g);
        tc_fence_after();
        uint32_t dp2[64];
        tmem_ld32(lane_base + 128 + (2 * hf) * 32, dp2);
        tmem_ld32(lane_base + 128 + (2 * hf + 1) * 32, dp2 + 32);
        tmem_ld_wait(dp2);
        tmem_ld_wait(dp2 + 32);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c = 2 * hf + cc;
          const uint32_t* dp = dp2 + 32 * cc;
          uint32_t pd[16];
#pragma unroll
          for (int i4 = 0; i4 < (USPB_DBG_NOCOMPUTE ? 0 : 8); ++i4) {
            const float4 D4 = lds_f4(vb + 512 + (c * 32 + 4 * i4) * 4);  // -delta of 4 q rows
            const float ndv[4] = {D4.x, D4.y, D4.z, D4.w};
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              // P^T as the dV MMA consumed it (bf16), widened
              const uint32_t w = pp2[cc][2 * i4 + e / 2];
              const float2 pw = make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
              const float2 d = fadd2(make_float2(__uint_as_float(dp[4 * i4 + e]), __uint_as_float(dp[4 * i4 + e + 1])),
                                     make_float2(ndv[e], ndv[e + 1]));
              const float2 ds = fmul2(pw, d);
              pd[2 * i4 + e / 2] = bwd_pack(ds.x, ds.y);
            }
          }
          st16(lane_base + 128 + packed_col(c), pd);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&ds_ready[USPB_DKDV_PAIRW ? cc : c]);
        }
        if (tr) bwd_trace(p, 4 * hf + 3, g);
      }
      // epilogue: warp half 0 stores dv (+)= dV, half 1 dk (+)= dK / sqrt(hs)
      const bool any = n > 0;
      if (any) {
        mbar_wait(acc_full, a_phase & 1);
        ++a_phase;
        tc_fence_after();
      }
      const bool valid = k_row < p.k_len;
      const size_t krow = (static_cast<size_t>(b) * p.k_len + (valid ? k_row : 0)) * p.kv_heads + kvh;
      if (hf == 0)
        store_rows<HS>(lane_base, 256, any, valid, p.dv + krow * HS, 1.f, p.accumulate != 0);
      else
        store_rows<HS>(lane_base, 256 + HS, any, valid, p.dk + krow * HS, p.inv_scale, p.accumulate != 0);
    }
  } else if (warp == C::kTmaWarp) {
    // ---------------------------------------------------- producer
    if (lane == 0) {
      uint32_t qd_it = 0, kv_it = 0;
      for (uint32_t it = 0;; ++it) {
        int u;
        if (!MC || crank == 0) {
          u = atomicAdd(&p.sched[0], 1);
          mbar_wait(u_empty, (it & 1) ^ 1);
          *reinterpret_cast<volatile int*>(unit_slot) = u;
          if constexpr (MC) {  // the same ticket to the peer CTA
            st_cluster_u32(mapa_shared(smem_u32(unit_slot), 1), static_cast<uint32_t>(u));
            mbar_arrive_cluster(mapa_shared(smem_u32(u_full), 1));
          }
          mbar_arrive(u_full);
        } else {  // MC peer: take the leader's ticket
          mbar_wait_cluster(u_full, it & 1);
          u = *reinterpret_cast<volatile int*>(unit_slot);
          mbar_arrive_cluster(mapa_shared(smem_u32(u_empty), 0));
        }
        if (u >= p.num_units) break;
        const uint32_t unit = p.units[u];
        const int kt = unit_ktile(unit), row = unit_row(unit), kvh = (unit >> 16) & 0xFF, b = unit >> 24;
        const int beg = p.tile_off[row], n = p.tile_off[row + 1] - beg;
        if (n == 0) continue;
        mbar_wait(kv_empty, (kv_it & 1) ^ 1);
        ++kv_it;
        mbar_arrive_expect_tx(kv_full, 2 * C::kTileBytes);
        for (int sb = 0; sb < C::kSub; ++sb) {
          tma_load_4d(sK + sb * C::kSubBytes, &p.tm_k, kv_full, sb * 64, kvh, kt * 128, b);
          tma_load_4d(sV + sb * C::kSubBytes, &p.tm_v, kv_full, sb * 64, kvh, kt * 128, b);
        }
        for (int gh = 0; gh < group; ++gh) {
          const int h = kvh * group + gh;
          for (int j = 0; j < n; ++j) {
            const int qt = p.tile_list[beg + j] & 0x7FFFFFFF;
            for (int which = 0; which < 2; ++which) {
              const uint32_t slot = qd_slot<NS>(qd_it);
              mbar_wait(&qd_empty[slot], ((qd_it / NS) & 1) ^ 1);
              bwd_trace(p, 14 + which, qd_it >> 1);
              ++qd_it;
              // QD1: Q, dO and the vector all complete on the Q slot's barrier
              // (the MMA warp then waits once per q tile)
              uint64_t* full = &qd_full[USPB_DKDV_QD1 && which == 1 ? qd_slot<NS>(qd_it - 2) : slot];
              if (!USPB_DKDV_QD1 || which == 0)
                mbar_arrive_expect_tx(full, (USPB_DKDV_QD1 ? 2 : 1) * C::kTileBytes + (which == 0 ? C::kVecBytes : 0));
              if (which == 0)
                bulk_g2s(vec + slot * C::kVecBytes,
                         p.qvec + ((static_cast<size_t>(b) * p.heads + h) * p.n_q_tiles + qt) * 384, C::kVecBytes,
                         full);
              const CUtensorMap* tm = which == 0 ? &p.tm_q : &p.tm_do;
              if constexpr (MC) {  // my half of the tile, to both CTAs
                tma_load_4d_mc(sQD + slot * C::kTileBytes + crank * C::kSubBytes, tm, full, int(crank) * 64, h,
                               qt * 128, b, uint16_t(0x3));
              } else {
                for (int sb = 0; sb < C::kSub; ++sb)
                  tma_load_4d(sQD + slot * C::kTileBytes + sb * C::kSubBytes, tm, full, sb * 64, h, qt * 128, b);
              }
            }
          }
        }
      }
      if (crank == 0 && atomicAdd(&p.sched[1], 1) == static_cast<int>(gridDim.x) / (MC ? 2 : 1) - 1) {
        p.sched[0] = 0;
        p.sched[1] = 0;
        __threadfence();
      }
    }
  } else if (warp == C::kMmaWarp) {
    // ---------------------------------------------------- MMA issue
    const uint64_t k_desc = smem_desc_sw128(smem_u32(sK), 16, 1024);
    const uint64_t v_desc = smem_desc_sw128(smem_u32(sV), 16, 1024);
    const uint64_t qd_desc0 = smem_desc_sw128(smem_u32(sQD), 16, 1024);
    const uint64_t qdmn_desc0 = smem_desc_sw128(smem_u32(sQD), C::kSubBytes, 1024);
    uint32_t qd_it = 0, kv_phase = 0, g = 0;
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it);
      if (u >= p.num_units) break;
      const int row = unit_row(p.units[u]);
      const int n = p.tile_off[row + 1] - p.tile_off[row];
      if (n == 0) continue;
      mbar_wait(kv_full, kv_phase & 1);
      ++kv_phase;
      tc_fence_after();
      const int total = group * n;
      auto ss = [&](uint32_t d, uint64_t ad, uint32_t slot) {  // D = A * B^T, B K-major from slot
        bwd_dispatch_slot<NS>(slot, [&](auto S) {
          constexpr int sl = decltype(S)::value;
          const uint64_t bd = qd_desc0 + static_cast<uint64_t>((sl * C::kTileBytes) >> 4);
          if (elect_one()) {
            if constexpr (HS == 128)
              mma_qk_hs128(d, ad, bd, C::kIdescSS, 0u);
            else
              mma_qk_hs64(d, ad, bd, C::kIdescSS, 0u);
          }
          __syncwarp();
        });
      };
      auto wait_qd = [&](uint32_t x) {
        if (USPB_DKDV_QD1 && (x & 1)) return;  // dO completed with its Q tile (waited before S)
        mbar_wait(&qd_full[qd_slot<NS>(x)], (x / NS) & 1);
        tc_fence_after();
      };
      // S^T(0) = K Q(0)^T, dP^T(0) = V dO(0)^T
      wait_qd(qd_it);
      ss(0, k_desc, qd_slot<NS>(qd_it));
      bwd_commit(s_full);
      wait_qd(qd_it + 1);
      ss(128, v_desc, qd_slot<NS>(qd_it + 1));
      bwd_commit(dp_full);
      for (int i = 0; i < total; ++i, ++g) {
        const uint32_t qi = qd_it + 2 * i, di = qi + 1;
        const uint64_t dbd = qdmn_desc0 + static_cast<uint64_t>(((qd_slot<NS>(di) * C::kTileBytes)) >> 4);
        const uint64_t qbd = qdmn_desc0 + static_cast<uint64_t>(((qd_slot<NS>(qi) * C::kTileBytes)) >> 4);
        const uint32_t acc = i > 0 ? 1u : 0u;
        // dV += P^T dO(i), chunk by chunk as P^T lands
#pragma unroll
        for (int n4 = 0; n4 < 4; ++n4) {
          const int c = chunk_at(n4);
          if (!USPB_DKDV_PAIRW || (n4 & 1) == 0) {
            mbar_wait(&p_ready[USPB_DKDV_PAIRW ? n4 >> 1 : c], g & 1);
            if (lane == 0) bwd_trace(p, 8 + (n4 >> 1), g);
            tc_fence_after();
          }
          if (elect_one())
            mma_ts_k2(256, packed_col(c), dbd + static_cast<uint64_t>(c * 256), C::kIdescTS, (acc | n4) ? 1u : 0u);
          __syncwarp();
        }
        // dO(i) is read by nothing after dV(i): release its slot now
        if constexpr (MC) {  // a slot is free once both CTAs' MMAs read it
          if (elect_one()) mma_commit_mc(&qd_empty[qd_slot<NS>(di)], uint16_t(0x3));
          __syncwarp();
        } else {
          bwd_commit(&qd_empty[qd_slot<NS>(di)]);
        }
        // S^T(i+1) over the S^T region (its P^T is consumed by the dV MMAs
        // issued above): overlaps this tile's dS^T work
        if (i + 1 < total) {
          wait_qd(qi + 2);
          ss(0, k_desc, qd_slot<NS>(qi + 2));
          bwd_commit(s_full);
          if (lane == 0) bwd_trace(p, 10, g);
        }
        // dK += dS^T Q(i), chunk by chunk as dS^T lands
#pragma unroll
        for (int n4 = 0; n4 < 4; ++n4) {
          const int c = chunk_at(n4);
          if (!USPB_DKDV_PAIRW || (n4 & 1) == 0) {
            mbar_wait(&ds_ready[USPB_DKDV_PAIRW ? n4 >> 1 : c], g & 1);
            if (lane == 0) bwd_trace(p, 11 + (n4 >> 1), g);
            tc_fence_after();
          }
          if (elect_one())
            mma_ts_k2(256 + HS, 128 + packed_col(c), qbd + static_cast<uint64_t>(c * 256), C::kIdescTS,
                      (acc | n4) ? 1u : 0u);
          __syncwarp();
        }
        // dP^T(i+1) over the dP^T region (its dS^T is consumed by the dK MMAs)
        if (i + 1 < total) {
          wait_qd(di + 2);
          ss(128, v_desc, qd_slot<NS>(di + 2));
          bwd_commit(dp_full);
          if (lane == 0) bwd_trace(p, 13, g);
        }
        if constexpr (MC) {
          if (elect_one()) mma_commit_mc(&qd_empty[qd_slot<NS>(qi)], uint16_t(0x3));
          __syncwarp();
        } else {
          bwd_commit(&qd_empty[qd_slot<NS>(qi)]);
        }
      }
      bwd_commit(acc_full);
      bwd_commit(kv_empty);
      qd_it += 2 * total;
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync();  // no remote traffic may target an exited CTA
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, 512);
}

// ============================================================ fused kernel
// One kernel for the whole block backward (attention_block_backward,
// attention.cpp:282-324): unit = (batch, kv head, 128-row key tile), loop
// over the visible q tiles (descending, see below) x the GQA group's q heads.
// Five GEMMs per (key tile, q tile) instead of the two-kernel path's seven:
//   S^T  = K Q^T            SS -> TMEM [0,128)
//   dP^T = V dO^T           SS -> TMEM [128,256)
//   dV  += P^T dO           TS (P^T bf16 over consumed S^T columns) -> [256,256+HS)
//   dQ   = dS K             SS, both MN-major -> TMEM [128,128+HS) (dP^T consumed)
//   dK  += dS^T Q           SS (dS^T K-major from shared memory) -> [256+HS,256+2HS)
// The compute warps store dS^T (bf16) once, into a 128B-swizzled shared tile
// — at head size 128 the slot of the tile's dO, dead once the dV MMAs
// completed; at 64 a buffer of its own — that serves as dK's K-major A and
// dQ's MN-major A. dQ(i) is a per-tile partial: four
// drain warps (one per TMEM lane quarter, thread = q row) read all of it into
// registers and release the dP region for dP^T(i+1), then stage it 32
// head-dim columns at a time (4 KB per warp, 128B-swizzled, double-buffered)
// in shared memory, from where TMA reduces it into the fp32 dQ rows
// (cp.reduce.async.bulk.tensor .add). Per-thread red.global.add from four
// warps sustains only ~14 B/clk/SM of the ~24 the L2 reduction path takes
// (tools/microbench/red_rate.cu) and set a 5.6k-clk tile period. With a
// key-tile pair per 2-CTA cluster (dQ pre-summed over DSMEM, or Q / dO
// shared by multicast) and with LSU row reductions it measured slower
// (DESIGN §4.3).
// q tiles are walked in descending order with the group's heads innermost, so
// the resident CTAs (consecutive key tiles of one kv head, longest first)
// work on the same q tile together (ascending, and heads rotated per key
// tile, measured the same at 32K and 128K). dQ accumulation order across key
// tiles is not fixed: the result is not bitwise reproducible run to run (the
// two-kernel path is). What bounds it (tools/trace_fused.py, round 2): the
// 64 KB of fp32 reductions per tile (~24 B/clk/SM through L2, measured) and
// the TMA unit they share with the Q / dO loads, whose 2-slot rings free a
// slot only when the tile's last MMA (dK) completes.
template <int HS>
struct FusedCfg {
  static_assert(HS == 128 || HS == 64, "the fused backward runs at kernel head size 64 or 128");
  static constexpr int kTileBytes = 128 * HS * 2;
  // dS^T (128 keys x 128 q, bf16 = 32 KB) fits over the tile's dO slot only
  // at head size 128; at 64 it gets its own buffer (released after dQ / dK)
  static constexpr bool kDsInDo = HS == 128;
  static constexpr int kDsBytes = 128 * 128 * 2;
  static constexpr int kSubBytes = 128 * 128;
  static constexpr int kSub = HS / 64;
  static constexpr int kCompute = 8, kDrain = 4;
  // 16 warps: 0-7 compute, 8-11 dQ drain (lane quarter = warp & 3), 12 TMA,
  // 13 MMA, 14-15 idle (complete the warpgroup for setmaxnreg). The drain
  // holds its q row's whole HS-column dQ partial in registers.
  static constexpr int kThreads = 512;
  static constexpr int kTmaWarp = 12, kMmaWarp = 13;
  static constexpr int kComputeRegs = 168, kDrainRegs = 144, kProducerRegs = 32;
  static_assert(2 * kComputeRegs + kDrainRegs + kProducerRegs <= 512, "register split (pool = 512 x 128)");
  static constexpr int kVecBytes = 2 * 128 * 4;  // -lse2 | -delta of one q tile
  static constexpr int kStageBytes = 32 * 32 * 4;  // fp32 dQ staging box: 32 rows x 32 columns, SW128
  static constexpr int kOffK = 0, kOffV = kTileBytes, kOffQ = 2 * kTileBytes, kOffDO = 4 * kTileBytes;
  static constexpr int kOffDS = 6 * kTileBytes;  // (HS = 64 only)
  static constexpr int kOffStage = kOffDS + (kDsInDo ? 0 : kDsBytes);
  static constexpr int kOffVec = kOffStage + 4 * 2 * kStageBytes;  // [warp][2]
  static constexpr int kOffBar = kOffVec + 2 * kVecBytes;
  static constexpr int kSmemBytes = kOffBar + 256;
  static_assert(kSmemBytes <= 232448, "fused smem");
  static constexpr uint32_t kIdescSS = idesc_bf16_f32(128, 128, 0, 0);  // S^T / dP^T
  static constexpr uint32_t kIdescTS = idesc_bf16_f32(128, HS, 0, 1);   // dV += P^T dO
  static constexpr uint32_t kIdescDK = idesc_bf16_f32(128, HS, 0, 1);   // dK += dS^T Q
  static constexpr uint32_t kIdescDQ = idesc_bf16_f32(128, HS, 1, 1);   // dQ = dS K
};

template <int HS>
__global__ void __launch_bounds__(FusedCfg<HS>::kThreads, 1) fa_bwd_fused_kernel(const __grid_constant__ BwdParams p) {
  using C = FusedCfg<HS>;
  constexpr uint32_t kS = 0, kDP = 128, kDV = 256, kDK = 256 + HS;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // the swizzled tiles need 1 KB alignment (no padding room)
  uint8_t* sK = smem + C::kOffK;
  uint8_t* sV = smem + C::kOffV;
  uint8_t* sQ = smem + C::kOffQ;    // [2]
  uint8_t* sDO = smem + C::kOffDO;  // [2]; HS 128: dS^T of tile g over dO(g) once dV(g) completed
  // the dS^T tile of the current q tile: dO's slot (HS 128) or its own buffer
  auto ds_base = [&](uint32_t slot) -> uint8_t* {
    return C::kDsInDo ? sDO + slot * C::kTileBytes : smem + C::kOffDS;
  };
  uint8_t* stage = smem + C::kOffStage;  // [drain warp][2] fp32 dQ boxes for the TMA reductions
  uint8_t* vec = smem + C::kOffVec;  // [2][-lse2 128 | -delta 128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* kv_full = bars + 0;
  uint64_t* kv_empty = bars + 1;
  uint64_t* q_full = bars + 2;    // [2] Q tile + its vector landed
  uint64_t* q_empty = bars + 4;   // [2] dK MMA of that tile done
  uint64_t* do_full = bars + 6;   // [2]
  uint64_t* do_empty = bars + 8;  // [2] dQ^T / dK MMAs (the last readers of the slot's dS^T) done
  uint64_t* s_full = bars + 10;
  uint64_t* p_ready = bars + 11;  // [2] P^T chunk pair in TMEM (256 arrivals)
  uint64_t* dp_full = bars + 13;
  uint64_t* ds_full = bars + 14;  // dS^T tile in shared memory (256 arrivals)
  uint64_t* dv_done = bars + 15;  // HS 128: dV MMAs done, the dO slot may take dS^T; HS 64: the dS^T buffer is free
  uint64_t* dq_full = bars + 16;  // dQ in TMEM
  uint64_t* dq_free = bars + 17;  // dQ read by the drain warps
  uint64_t* acc_full = bars + 18;
  uint64_t* u_full = bars + 19;
  uint64_t* u_empty = bars + 20;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 21);
  int* unit_slot = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&do_full[s], 1);
      mbar_init(&do_empty[s], 1);
      mbar_init(&p_ready[s], 256);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 256);
    mbar_init(dv_done, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, C::kDrain);
    mbar_init(acc_full, 1);
    mbar_init(u_full, 1);
    mbar_init(u_empty, C::kCompute + C::kDrain + 1);  // compute + drain + MMA warps
    fence_barrier_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tmem != 0) __trap();
  const int group = p.heads / p.kv_heads;

  auto get_unit = [&](uint32_t it) {
    mbar_wait(u_full, it & 1);
    const int u = *reinterpret_cast<volatile int*>(unit_slot);
    __syncwarp();
    if (lane == 0) mbar_arrive(u_empty);
    return u;
  };
  // tile i of a unit with n q tiles: q tiles descending, heads innermost
  auto tile_entry = [&](int beg, int n, int i) { return p.tile_list[beg + (n - 1 - i / group)]; };
  auto tile_head = [&](int kvh, int i) { return kvh * group + i % group; };

  if (warp >= C::kCompute + C::kDrain) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::kProducerRegs));
  } else if (warp >= C::kCompute) {
    static_assert(C::kDrainRegs >= 128, "drain warps grow from the launch's 128");
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::kDrainRegs));
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::kComputeRegs));
  }

  if (warp < C::kCompute) {
    // ---------------------------------------------------- compute warps (thread = key row)
    const int q4 = warp & 3, hf = warp >> 2;
    const int key_in_tile = q4 * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const float sl2 = p.scale_log2;
    const uint32_t vec_s = smem_u32(vec);
    // this thread's row of the dS^T tile: 64-column block hf, 128-byte row
    // key_in_tile, 16-byte units XOR-swizzled by the row (SWIZZLE_128B)
    const float isc = p.inv_scale;
    const uint32_t ds_row0 = smem_u32(ds_base(0)) + hf * C::kSubBytes + key_in_tile * 128;
    const uint32_t swz = static_cast<uint32_t>(key_in_tile & 7);
    uint32_t g = 0, a_phase = 0;
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it);
      if (u >= p.num_units) break;
      const uint32_t unit = p.units[u];
      const int kt = unit & 0xFFFF, kvh = (unit >> 16) & 0xFF, b = unit >> 24;
      const int beg = p.tile_off[kt], n = p.tile_off[kt + 1] - beg;
      const int k_row = kt * 128 + key_in_tile;
      const int kpos = p.k_pos[k_row];
      const int total = group * n;
      for (int i = 0; i < total; ++i, ++g) {
        const int entry = tile_entry(beg, n, i);
        const int qt = entry & 0x7FFFFFFF;
        const uint32_t s = g & 1u;
        mbar_wait(&q_full[s], (g >> 1) & 1);  // this q tile's -lse2 / -delta came with its Q tile
        const uint32_t vb = vec_s + s * C::kVecBytes;
        // phase 1: P^T = exp2(S^T * scale - lse2), packed over consumed S^T columns
        const bool tr = q4 == 0 && lane == 0;
        // the first chunk's -lse2 values (32 q columns, broadcast reads)
        // issued before the S^T wait so their latency hides behind it: the
        // compute warps stalled on these loads (ncu short-scoreboard);
        // +5.5 % (981 -> 1035 TFLOP/s at 128K, A/B). All 64 columns spill.
        float4 lv[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) lv[x] = lds_f4(vb + (hf * 64 + 4 * x) * 4);
        mbar_wait(s_full, g & 1);
        if (tr && hf == 0) bwd_trace(p, 0, g);
        tc_fence_after();
        uint32_t pp2[2][16];
        uint32_t sv2[64];
        tmem_ld32(lane_base + kS + (2 * hf) * 32, sv2);
        tmem_ld32(lane_base + kS + (2 * hf + 1) * 32, sv2 + 32);
        tmem_ld_wait(sv2);
        tmem_ld_wait(sv2 + 32);
        auto p_chunks = [&](auto masked) {
          constexpr bool kMasked = decltype(masked)::value;
          float4 lv1[8];
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = 2 * hf + cc;
            const uint32_t* sv = sv2 + 32 * cc;
            uint32_t* pp = pp2[cc];
#pragma unroll
            for (int i4 = 0; i4 < 8; ++i4) {
              const float4 L4 = cc == 0 ? lv[i4] : lv1[i4];
              const float2 x01 = ffma2(make_float2(__uint_as_float(sv[4 * i4]), __uint_as_float(sv[4 * i4 + 1])),
                                       make_float2(sl2, sl2), make_float2(L4.x, L4.y));
              const float2 x23 = ffma2(make_float2(__uint_as_float(sv[4 * i4 + 2]), __uint_as_float(sv[4 * i4 + 3])),
                                       make_float2(sl2, sl2), make_float2(L4.z, L4.w));
              float pv[4] = {ex2(x01.x), ex2(x01.y), ex2(x23.x), ex2(x23.y)};
              if constexpr (kMasked) {
                const int4 qv = __ldg(reinterpret_cast<const int4*>(p.q_pos + qt * 128 + c * 32) + i4);
                pv[0] = kpos > qv.x ? 0.f : pv[0];
                pv[1] = kpos > qv.y ? 0.f : pv[1];
                pv[2] = kpos > qv.z ? 0.f : pv[2];
                pv[3] = kpos > qv.w ? 0.f : pv[3];
              }
              pp[2 * i4] = bwd_pack(pv[0], pv[1]);
              pp[2 * i4 + 1] = bwd_pack(pv[2], pv[3]);
            }
            if (cc == 0) {  // the second chunk's -lse2 while the first chunk's P^T is stored
#pragma unroll
              for (int x = 0; x < 8; ++x) lv1[x] = lds_f4(vb + (hf * 64 + 32 + 4 * x) * 4);
            }
            st16(lane_base + kS + packed_col(c), pp);
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_ready[cc]);
          }
        };
        if (entry < 0)
          p_chunks(std::true_type{});
        else
          p_chunks(std::false_type{});
        if (tr) bwd_trace(p, 4 * hf + 1, g);
        // phase 2: dS^T = P^T (dP^T - delta) -> the shared dS^T tile
        float4 dv4[8];  // -delta / sqrt(hs) of the first chunk's 32 q columns, before the dP^T wait
#pragma unroll
        for (int x = 0; x < 8; ++x) dv4[x] = lds_f4(vb + 512 + (hf * 64 + 4 * x) * 4);
        mbar_wait(dp_full, g & 1);
        if (tr) bwd_trace(p, 4 * hf + 2, g);
        tc_fence_after();
        uint32_t dp2[64];
        tmem_ld32(lane_base + kDP + (2 * hf) * 32, dp2);
        tmem_ld32(lane_base + kDP + (2 * hf + 1) * 32, dp2 + 32);
        tmem_ld_wait(dp2);
        tmem_ld_wait(dp2 + 32);
        uint32_t pd2[2][16];
        float4 dv1[8];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const uint32_t* dp = dp2 + 32 * cc;
          uint32_t* pd = pd2[cc];
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4) {
            const float4 D4 = cc == 0 ? dv4[i4] : dv1[i4];  // -delta / sqrt(hs)
            const float ndv[4] = {D4.x, D4.y, D4.z, D4.w};
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              const uint32_t w = pp2[cc][2 * i4 + e / 2];
              const float2 pw = make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
              // (dP - delta) / sqrt(hs): ds carries the scale (attention.cpp's
              // ds = p (dp - delta) / sqrt(hs)), so neither dQ nor dK is rescaled
              const float2 d = ffma2(make_float2(__uint_as_float(dp[4 * i4 + e]), __uint_as_float(dp[4 * i4 + e + 1])),
                                     make_float2(isc, isc), make_float2(ndv[e], ndv[e + 1]));
              const float2 ds = fmul2(pw, d);
              pd[2 * i4 + e / 2] = bwd_pack(ds.x, ds.y);
            }
          }
          if (cc == 0) {
#pragma unroll
            for (int x = 0; x < 8; ++x) dv1[x] = lds_f4(vb + 512 + (hf * 64 + 32 + 4 * x) * 4);
          }
        }
        if (tr && hf == 0) bwd_trace(p, 12, g);
        // HS 128: dS^T(g) goes over dO(g), once the dV MMAs have read it;
        // HS 64: into the dS^T buffer, once the previous tile's dQ / dK read it
        if (C::kDsInDo)
          mbar_wait(dv_done, g & 1);
        else if (g > 0)
          mbar_wait(dv_done, (g - 1) & 1);
        if (tr && hf == 0) bwd_trace(p, 4, g);
        const uint32_t ds_row = ds_row0 + (C::kDsInDo ? s * C::kTileBytes : 0u);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t unit16 = static_cast<uint32_t>(cc * 4 + k) ^ swz;
            sts_v4(ds_row + unit16 * 16, pd2[cc][4 * k], pd2[cc][4 * k + 1], pd2[cc][4 * k + 2], pd2[cc][4 * k + 3]);
          }
        fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
        tc_fence_before();
        mbar_arrive(ds_full);
        if (tr) bwd_trace(p, 4 * hf + 3, g);
      }
      // epilogue: warp half 0 stores dv (+)= dV, half 1 dk (+)= dK / sqrt(hs)
      const bool any = n > 0;
      if (any) {
        mbar_wait(acc_full, a_phase & 1);
        ++a_phase;
        tc_fence_after();
      }
      const bool valid = k_row < p.k_len;
      const size_t krow = (static_cast<size_t>(b) * p.k_len + (valid ? k_row : 0)) * p.kv_heads + kvh;
      if (hf == 0)
        store_rows<HS>(lane_base, kDV, any, valid, p.dv + krow * HS, 1.f, p.accumulate != 0);
      else
        store_rows<HS>(lane_base, kDK, any, valid, p.dk + krow * HS, 1.f, p.accumulate != 0);
    }
  } else if (warp < C::kCompute + C::kDrain) {
    // ---------------------------------------------------- dQ drain (thread = q row)
    const int q4 = warp & 3;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + kDP;
    // this warp's two 4 KB staging boxes; this thread's 128-byte row in them
    const uint32_t st_row = smem_u32(stage) + q4 * 2 * C::kStageBytes + lane * 128;
    const uint32_t swz = static_cast<uint32_t>(lane & 7);
    uint32_t g = 0, chunk = 0;
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it);
      if (u >= p.num_units) break;
      const uint32_t unit = p.units[u];
      const int kt = unit & 0xFFFF, kvh = (unit >> 16) & 0xFF, b = unit >> 24;
      const int beg = p.tile_off[kt], n = p.tile_off[kt + 1] - beg;
      const int total = group * n;
      for (int i = 0; i < total; ++i, ++g) {
        const int qt = tile_entry(beg, n, i) & 0x7FFFFFFF;
        const int h = tile_head(kvh, i);
        mbar_wait(dq_full, g & 1);
        if (q4 == 0 && lane == 0) bwd_trace(p, 14, g);
        tc_fence_after();
        // this q row's whole dQ partial into registers, then release the dP
        // region: staging and reduction run behind dP^T(i+1)
        uint32_t r[HS];
#pragma unroll
        for (int c = 0; c < HS / 32; ++c) tmem_ld32(lane_base + 32 * c, r + 32 * c);
#pragma unroll
        for (int c = 0; c < HS / 32; ++c) tmem_ld_wait(r + 32 * c);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dq_free);  // the dP region may take dP^T(i+1)
#pragma unroll
        for (int cb = 0; cb < HS / 32; ++cb, ++chunk) {
          const uint32_t buf = chunk & 1u;
          // the box was last read by the reduction issued two chunks ago
          // (USPB_FUSED_RDEPTH = reductions a warp keeps queued on the TMA
          // unit, which the Q / dO loads queue behind)
          if (lane == 0) bulk_wait_group_read<USPB_FUSED_RDEPTH>();
          __syncwarp();
          const uint32_t row = st_row + buf * C::kStageBytes;
#pragma unroll
          for (int k = 0; k < 8; ++k)  // 16-byte units XOR-swizzled by the row (SWIZZLE_128B)
            sts_v4(row + ((static_cast<uint32_t>(k) ^ swz) << 4), r[32 * cb + 4 * k], r[32 * cb + 4 * k + 1],
                   r[32 * cb + 4 * k + 2], r[32 * cb + 4 * k + 3]);
          fence_proxy_async_smem();  // generic-proxy stores -> visible to the TMA unit
          __syncwarp();
          if (lane == 0) {
            // dq[b][32 rows of this warp][h][32 cb ..] += the box (rows past
            // q_len are dropped by the tensor map bounds)
            if (!USPB_FUSED_NORED)
              tma_reduce_add_4d(&p.tm_dq, stage + (q4 * 2 + buf) * C::kStageBytes, 32 * cb, h,
                                qt * 128 + 32 * q4, b);
            bulk_commit_group();
          }
        }
        if (q4 == 0 && lane == 0) bwd_trace(p, 15, g);  // all chunks handed to TMA
      }
    }
    if (lane == 0) bulk_wait_group<0>();  // every reduction has landed before the CTA exits
  } else if (warp == C::kTmaWarp) {
    // ---------------------------------------------------- producer
    if (lane == 0) {
      uint32_t g = 0, kv_it = 0;
      for (uint32_t it = 0;; ++it) {
        const int u = atomicAdd(&p.sched[0], 1);
        mbar_wait(u_empty, (it & 1) ^ 1);
        *reinterpret_cast<volatile int*>(unit_slot) = u;
        mbar_arrive(u_full);
        if (u >= p.num_units) break;
        const uint32_t unit = p.units[u];
        const int kt = unit & 0xFFFF, kvh = (unit >> 16) & 0xFF, b = unit >> 24;
        const int beg = p.tile_off[kt], n = p.tile_off[kt + 1] - beg;
        if (n == 0) continue;
        mbar_wait(kv_empty, (kv_it & 1) ^ 1);
        ++kv_it;
        mbar_arrive_expect_tx(kv_full, 2 * C::kTileBytes);
        for (int sb = 0; sb < C::kSub; ++sb) {
          tma_load_4d(sK + sb * C::kSubBytes, &p.tm_k, kv_full, sb * 64, kvh, kt * 128, b);
          tma_load_4d(sV + sb * C::kSubBytes, &p.tm_v, kv_full, sb * 64, kvh, kt * 128, b);
        }
        const int total = group * n;
        for (int i = 0; i < total; ++i, ++g) {
          const int qt = tile_entry(beg, n, i) & 0x7FFFFFFF;
          const int h = tile_head(kvh, i);
          const uint32_t s = g & 1u, ph = ((g >> 1) & 1) ^ 1;
          mbar_wait(&q_empty[s], ph);
          mbar_arrive_expect_tx(&q_full[s], C::kTileBytes + C::kVecBytes);
          bulk_g2s(vec + s * C::kVecBytes, p.qvec + ((static_cast<size_t>(b) * p.heads + h) * p.n_q_tiles + qt) * 384,
                   C::kVecBytes, &q_full[s]);
          for (int sb = 0; sb < C::kSub; ++sb)
            tma_load_4d(sQ + s * C::kTileBytes + sb * C::kSubBytes, &p.tm_q, &q_full[s], sb * 64, h, qt * 128, b);
          mbar_wait(&do_empty[s], ph);
          mbar_arrive_expect_tx(&do_full[s], C::kTileBytes);
          for (int sb = 0; sb < C::kSub; ++sb)
            tma_load_4d(sDO + s * C::kTileBytes + sb * C::kSubBytes, &p.tm_do, &do_full[s], sb * 64, h, qt * 128, b);
        }
      }
      if (atomicAdd(&p.sched[1], 1) == static_cast<int>(gridDim.x) - 1) {
        p.sched[0] = 0;
        p.sched[1] = 0;
        __threadfence();
      }
    }
  } else if (warp == C::kMmaWarp) {
    // ---------------------------------------------------- MMA issue
    const uint64_t k_desc = smem_desc_sw128(smem_u32(sK), 16, 1024);
    const uint64_t v_desc = smem_desc_sw128(smem_u32(sV), 16, 1024);
    const uint64_t q_desc0 = smem_desc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t do_desc0 = smem_desc_sw128(smem_u32(sDO), 16, 1024);
    const uint64_t q_mn0 = smem_desc_sw128(smem_u32(sQ), C::kSubBytes, 1024);
    const uint64_t do_mn0 = smem_desc_sw128(smem_u32(sDO), C::kSubBytes, 1024);
    const uint64_t k_mn = smem_desc_sw128(smem_u32(sK), C::kSubBytes, 1024);
    constexpr uint64_t kSlot = C::kTileBytes >> 4;  // descriptor units per ring slot
    // the dS^T tile as dQ's MN-major A and dK's K-major A (HS 64: its own buffer)
    const uint64_t ds_mn0 = C::kDsInDo ? do_mn0 : smem_desc_sw128(smem_u32(smem + C::kOffDS), C::kSubBytes, 1024);
    const uint64_t ds_k0 = C::kDsInDo ? do_desc0 : smem_desc_sw128(smem_u32(smem + C::kOffDS), 16, 1024);
    constexpr uint64_t kDsSlot = C::kDsInDo ? kSlot : 0;
    auto qk = [&](uint32_t d, uint64_t ad, uint64_t bd) {  // D = A B^T over the head dimension
      if (elect_one()) {
        if constexpr (HS == 128)
          mma_qk_hs128(d, ad, bd, C::kIdescSS, 0u);
        else
          mma_qk_hs64(d, ad, bd, C::kIdescSS, 0u);
      }
      __syncwarp();
    };
    uint32_t g = 0, kv_phase = 0;
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it);
      if (u >= p.num_units) break;
      const int kt = p.units[u] & 0xFFFF;
      const int n = p.tile_off[kt + 1] - p.tile_off[kt];
      if (n == 0) continue;
      const int total = group * n;
      mbar_wait(kv_full, kv_phase & 1);
      ++kv_phase;
      tc_fence_after();
      // prologue: S^T, dP^T of the unit's first tile
      {
        const uint32_t s = g & 1u;
        mbar_wait(&q_full[s], (g >> 1) & 1);
        tc_fence_after();
        qk(kS, k_desc, q_desc0 + s * kSlot);
        bwd_commit(s_full);
        if (g > 0) mbar_wait(dq_free, (g - 1) & 1);  // the previous tile's dQ^T left the dP region
        mbar_wait(&do_full[s], (g >> 1) & 1);
        tc_fence_after();
        qk(kDP, v_desc, do_desc0 + s * kSlot);
        bwd_commit(dp_full);
      }
      for (int i = 0; i < total; ++i, ++g) {
        const uint32_t s = g & 1u, s1 = s ^ 1u, ph1 = ((g + 1) >> 1) & 1;
        // dV += P^T dO(g), per chunk pair as P^T lands
        const uint64_t dob = do_mn0 + s * kSlot;
#pragma unroll
        for (int n4 = 0; n4 < 4; ++n4) {
          const int c = chunk_at(n4);
          if ((n4 & 1) == 0) {
            mbar_wait(&p_ready[n4 >> 1], g & 1);
            if (n4 == 2 && lane == 0) bwd_trace(p, 8, g);
            tc_fence_after();
          }
          if (elect_one())
            mma_ts_k2(kDV, kS + packed_col(c), dob + static_cast<uint64_t>(c * 256), C::kIdescTS,
                      (i > 0 || n4 > 0) ? 1u : 0u);
          __syncwarp();
        }
        if constexpr (C::kDsInDo) {
          bwd_commit(dv_done);  // dO(g) consumed: the compute warps may write dS^T(g) over it
        } else {
          bwd_commit(&do_empty[s]);  // dO(g) consumed (dS^T has its own buffer)
        }
        // S^T(g+1) over the S region (P^T(g) is read by the dV MMAs above),
        // and dQ(g) into the dP region then dK(g) once dS^T(g) is in shared
        // memory: whichever is ready first is issued first. Q(g+1) is
        // loaded only once dK(g-1) completed (two Q slots), so waiting for it
        // before dQ(g) / dK(g) would also delay dK(g) and with it Q(g+2).
        auto issue_s_next = [&] {
          tc_fence_after();
          qk(kS, k_desc, q_desc0 + s1 * kSlot);
          bwd_commit(s_full);
          if (lane == 0) bwd_trace(p, 9, g);
        };
        auto issue_dq_dk = [&] {
          if (lane == 0) bwd_trace(p, 10, g);
          tc_fence_after();
          if (elect_one()) mma_mn_mn_chain(kDP, ds_mn0 + s * kDsSlot, k_mn, C::kIdescDQ, 0u);  // A = dS, B = K
          __syncwarp();
          bwd_commit(dq_full);
          if (elect_one())
            mma_kmaj_mn_chain(kDK, ds_k0 + s * kDsSlot, q_mn0 + s * kSlot, C::kIdescDK, i > 0 ? 1u : 0u);
          __syncwarp();
          bwd_commit(&q_empty[s]);
          if constexpr (C::kDsInDo)
            bwd_commit(&do_empty[s]);  // the slot's dS^T has been read
          else
            bwd_commit(dv_done);  // the dS^T buffer has been read
          if (lane == 0) bwd_trace(p, 11, g);
        };
        if (!USPB_FUSED_DYN || i + 1 >= total) {
          if (i + 1 < total) {
            mbar_wait(&q_full[s1], ph1);
            issue_s_next();
          }
          mbar_wait(ds_full, g & 1);
          issue_dq_dk();
        } else {
          bool s_done = false, d_done = false;
          uint32_t spins = 0;
          while (!(s_done && d_done)) {
            if (!s_done && mbar_test(&q_full[s1], ph1)) {
              issue_s_next();
              s_done = true;
            } else if (!d_done && mbar_test(ds_full, g & 1)) {
              issue_dq_dk();
              d_done = true;
            } else if (++spins == (1u << 28)) {
              __trap();  // a pipeline deadlock fails the launch instead of hanging
            }
          }
        }
        // dP^T(g+1) once the drain warps have read dQ^T(g)
        if (i + 1 < total) {
          mbar_wait(dq_free, g & 1);
          mbar_wait(&do_full[s1], ph1);
          tc_fence_after();
          qk(kDP, v_desc, do_desc0 + s1 * kSlot);
          bwd_commit(dp_full);
          if (lane == 0) bwd_trace(p, 13, g);
        }
      }
      bwd_commit(acc_full);
      bwd_commit(kv_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, 512);
}

// ============================================================ small kernels
__global__ void delta_kernel(const uint16_t* o, const uint16_t* dout, float* delta, int64_t batch, int64_t q_len,
                             int heads, int hs, int64_t n_qt, const float* lse, const int32_t* q_pos, float* qvec,
                             float delta_scale) {
  // one warp per row (b, t, h) over the padded rows t < n_qt * 128: 16-byte
  // loads, fp32 dot, shuffle reduction
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t t_pad = n_qt * 128;
  if (row >= batch * t_pad * heads) return;
  const int h = static_cast<int>(row % heads);
  const int64_t t = (row / heads) % t_pad, b = row / (heads * t_pad);
  const bool valid = t < q_len;
  float acc = 0.f;
  const int64_t r = (b * q_len + (valid ? t : 0)) * heads + h;
  if (valid) {
    const uint16_t* a = o + r * hs;
    const uint16_t* bq = dout + r * hs;
    for (int e = lane * 2; e < hs; e += 64) {
      const uint32_t x = *reinterpret_cast<const uint32_t*>(a + e);
      const uint32_t y = *reinterpret_cast<const uint32_t*>(bq + e);
      acc = fmaf(__uint_as_float(x << 16), __uint_as_float(y << 16), acc);
      acc = fmaf(__uint_as_float(x & 0xFFFF0000u), __uint_as_float(y & 0xFFFF0000u), acc);
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  }
  if (lane == 0) {
    if (valid) delta[r] = acc;
    if (qvec) {
      float* v = qvec + ((b * heads + h) * n_qt + t / 128) * 384 + (t % 128);
      // negated, for the dK/dV kernel's packed FFMA2 / FADD2
      v[0] = valid ? -(lse[r] * 1.4426950408889634f) : -INFINITY;  // padding rows: p = 0
      v[128] = valid ? -acc * delta_scale : -0.f;
      v[256] = __int_as_float(q_pos[t]);
    }
  }
}

__global__ void cast_rows_kernel(const float* src, const float* src2, uint16_t* dst, int64_t rows, int hs_src,
                                 int hs_dst) {
  const int64_t total = rows * hs_dst;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / hs_dst, c = i % hs_dst;
    float v = src[r * hs_src + c];
    if (src2) v += src2[r * hs_src + c];
    uint32_t bits = __float_as_uint(v);
    bits += 0x7FFFu + ((bits >> 16) & 1u);  // round to nearest even
    dst[i] = static_cast<uint16_t>(bits >> 16);
  }
}


}  // namespace

template <int HS, int MC>
static cudaError_t launch_dq_impl(const BwdParams& p, int grid, cudaStream_t stream) {
  using C = BwdCfg<HS>;
  auto kern = fa_bwd_dq_kernel<HS, MC>;
  static std::atomic<uint64_t> done{0};
  const cudaError_t once = ensure_smem_attr(kern, C::kDqSmemBytes, done);
  if (once != cudaSuccess) return once;
  if constexpr (MC) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid & ~1), 1, 1);
    cfg.blockDim = dim3(C::kThreads, 1, 1);
    cfg.dynamicSmemBytes = C::kDqSmemBytes;
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
  kern<<<grid, C::kThreads, C::kDqSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_bwd_dq(const BwdParams& p, int hs, int grid, cudaStream_t stream) {
  if (hs == 128) return p.cluster ? launch_dq_impl<128, 1>(p, grid, stream) : launch_dq_impl<128, 0>(p, grid, stream);
  if (hs == 64 && !p.cluster) return launch_dq_impl<64, 0>(p, grid, stream);
  return cudaErrorInvalidValue;
}

template <int HS, int MC>
static cudaError_t launch_dkdv_impl(const BwdParams& p, int grid, cudaStream_t stream) {
  using C = BwdCfg<HS>;
  auto kern = fa_bwd_dkdv_kernel<HS, MC>;
  static std::atomic<uint64_t> done{0};
  const cudaError_t once = ensure_smem_attr(kern, C::kSmemBytes, done);
  if (once != cudaSuccess) return once;
  if constexpr (MC) {
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

cudaError_t launch_bwd_dkdv(const BwdParams& p, int hs, int grid, cudaStream_t stream) {
  if (hs == 128)
    return p.cluster ? launch_dkdv_impl<128, 1>(p, grid, stream) : launch_dkdv_impl<128, 0>(p, grid, stream);
  if (hs == 64 && !p.cluster) return launch_dkdv_impl<64, 0>(p, grid, stream);
  return cudaErrorInvalidValue;
}

template <int HS>
static cudaError_t launch_fused_impl(const BwdParams& p, int grid, cudaStream_t stream) {
  using C = FusedCfg<HS>;
  auto kern = fa_bwd_fused_kernel<HS>;
  static std::atomic<uint64_t> done{0};
  const cudaError_t once = ensure_smem_attr(kern, C::kSmemBytes, done);
  if (once != cudaSuccess) return once;
  kern<<<grid, C::kThreads, C::kSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_bwd_fused(const BwdParams& p, int hs, int grid, cudaStream_t stream) {
  if (hs == 128) return launch_fused_impl<128>(p, grid, stream);
  if (hs == 64) return launch_fused_impl<64>(p, grid, stream);
  return cudaErrorInvalidValue;
}

cudaError_t launch_bwd_delta(const void* o, const void* dout, float* delta, int64_t batch, int64_t q_len,
                             int heads, int hs, const float* lse, const int32_t* q_pos, float* qvec,
                             float qvec_delta_scale, cudaStream_t stream) {
  const int64_t n_qt = (q_len + 127) / 128;
  const int64_t rows = batch * n_qt * 128 * heads;
  if (rows == 0) return cudaSuccess;
  const int64_t threads = rows * 32;
  const int grid = static_cast<int>((threads + 255) / 256);
  delta_kernel<<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(o), static_cast<const uint16_t*>(dout), delta,
                                         batch, q_len, heads, hs, n_qt, lse, q_pos, qvec, qvec_delta_scale);
  return cudaGetLastError();
}

__global__ void add_f32_kernel(const float4* a, float4* acc, int64_t n4) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 x = a[i];
    float4 y = acc[i];
    y.x = x.x + y.x;
    y.y = x.y + y.y;
    y.z = x.z + y.z;
    y.w = x.w + y.w;
    acc[i] = y;
  }
}

cudaError_t launch_add_f32(const float* blk, float* acc, int64_t n, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (n % 4 != 0) return cudaErrorInvalidValue;
  const int64_t n4 = n / 4;
  const int64_t blocks = (n4 + 255) / 256;
  add_f32_kernel<<<static_cast<int>(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, stream>>>(
      reinterpret_cast<const float4*>(blk), reinterpret_cast<float4*>(acc), n4);
  return cudaGetLastError();
}

cudaError_t launch_cast_rows(const float* src, const float* src2, void* dst, int64_t rows, int hs_src,
                             int hs_dst, cudaStream_t stream) {
  const int64_t total = rows * hs_dst;
  if (total == 0) return cudaSuccess;
  const int64_t blocks = (total + 255) / 256;
  const int grid = static_cast<int>(blocks < 148 * 16 ? blocks : 148 * 16);
  cast_rows_kernel<<<grid, 256, 0, stream>>>(src, src2, static_cast<uint16_t*>(dst), rows, hs_src, hs_dst);
  return cudaGetLastError();
}

}  // namespace uspb200
