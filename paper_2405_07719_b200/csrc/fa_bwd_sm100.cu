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

__device__ __forceinline__ void bwd_commit(uint64_t* bar) {
  if (elect_one()) mma_commit(bar);
  __syncwarp();
}

__device__ __forceinline__ void bwd_bar_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int HS>
struct BwdCfg {
  static constexpr int kTile = 128;
  static constexpr int kTileBytes = kTile * HS * 2;  // one 128-row bf16 tile
  static constexpr int kSubBytes = 128 * 128;
  static constexpr int kSub = HS / 64;
  static constexpr int kThreads = 192;  // 4 compute warps, TMA warp, MMA warp
  static constexpr int kTmaWarp = 4, kMmaWarp = 5;
  static constexpr int kBudget = 227 * 1024 - 4096;
  static constexpr int kStages = (kBudget - 2 * kTileBytes) / kTileBytes > 6
                                     ? 6
                                     : (kBudget - 2 * kTileBytes) / kTileBytes;
  static constexpr int kSmemBytes = 1024 + 2 * kTileBytes + kStages * kTileBytes + 4096;
  static constexpr uint32_t kIdescSS = idesc_bf16_f32(128, 128, 0, 0);  // S / dP
  static constexpr uint32_t kIdescTS = idesc_bf16_f32(128, HS, 0, 1);   // acc += X^T-style
  static_assert(kStages >= 2, "smem");
};

// ============================================================ dq kernel
// TMEM: S [0,128) (dS bf16 over its first 64 columns), dP [128,256),
// dQ [256, 256+HS).
template <int HS>
__global__ void __launch_bounds__(BwdCfg<HS>::kThreads, 1) fa_bwd_dq_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdCfg<HS>;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sDO = smem + C::kTileBytes;
  uint8_t* sKV = smem + 2 * C::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + NS * C::kTileBytes);
  uint64_t* q_full = bars;           // Q + dO landed
  uint64_t* q_empty = bars + 1;
  uint64_t* s_full = bars + 2;       // S and dP in TMEM
  uint64_t* ds_ready = bars + 3;     // dS written (128 arrivals)
  uint64_t* dq_full = bars + 4;      // unit's last dQ MMA done
  uint64_t* kv_full = bars + 5;      // [NS]
  uint64_t* kv_empty = kv_full + NS; // [NS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_empty + NS);
  int* unit_slot = reinterpret_cast<int*>(tmem_slot + 2);
  uint64_t* u_full = reinterpret_cast<uint64_t*>(unit_slot + 2);
  uint64_t* u_empty = u_full + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(ds_ready, 128);
    mbar_init(dq_full, 1);
    mbar_init(u_full, 1);
    mbar_init(u_empty, 5);  // 4 compute warps + MMA warp
    for (int s = 0; s < NS; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tmem != 0) __trap();
  const int group = p.heads / p.kv_heads;

  // unit ticket hand-off: producer claims, consumers read (depth 1)
  auto get_unit = [&](uint32_t it, bool whole_warp) {
    mbar_wait(u_full, it & 1);
    const int u = *reinterpret_cast<volatile int*>(unit_slot);
    if (whole_warp) {
      __syncwarp();
      if (lane == 0) mbar_arrive(u_empty);
    } else {
      mbar_arrive(u_empty);
    }
    return u;
  };

  if (warp < 4) {
    // ---------------------------------------------------- compute warps
    const int row_in_tile = warp * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const float sl2 = p.scale_log2;
    uint32_t s_phase = 0, d_phase = 0;
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it, true);
      if (u >= p.num_units) break;
      const uint32_t unit = p.units[u];
      const int qt = unit & 0xFFFF, h = (unit >> 16) & 0xFF, b = unit >> 24;
      const int beg = p.tile_off[qt], n = p.tile_off[qt + 1] - beg;
      const int q_row = qt * 128 + row_in_tile;
      const bool valid = q_row < p.q_len;
      const size_t row = (static_cast<size_t>(b) * p.q_len + (valid ? q_row : 0)) * p.heads + h;
      const float lse2 = valid ? p.lse[row] * 1.4426950408889634f : 0.f;
      const float dlt = valid ? p.delta[row] : 0.f;
      const int qpos = p.q_pos[q_row];
      for (int j = 0; j < n; ++j) {
        const int entry = p.tile_list[beg + j];
        mbar_wait(s_full, s_phase & 1);
        ++s_phase;
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t s[32], dp[32];
          tmem_ld32(lane_base + c * 32, s);
          tmem_ld32(lane_base + 128 + c * 32, dp);
          tmem_ld_wait(s);
          tmem_ld_wait(dp);
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
          for (int i = 0; i < 16; ++i) {
            const float p0 = ex2(fmaf(__uint_as_float(s[2 * i]), sl2, -lse2));
            const float p1 = ex2(fmaf(__uint_as_float(s[2 * i + 1]), sl2, -lse2));
            const float d0 = p0 * (__uint_as_float(dp[2 * i]) - dlt);
            const float d1 = p1 * (__uint_as_float(dp[2 * i + 1]) - dlt);
            pk[i] = pack_bf16x2(d0, d1);
          }
          // dS chunk c -> S columns [16c, 16c+16): already consumed
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
              "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(lane_base + c * 16),
              "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]),
              "r"(pk[7]), "r"(pk[8]), "r"(pk[9]), "r"(pk[10]), "r"(pk[11]), "r"(pk[12]), "r"(pk[13]),
              "r"(pk[14]), "r"(pk[15])
              : "memory");
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(ds_ready);
      }
      // epilogue: dq (+)= dQ / sqrt(hs)
      if (n > 0) {
        mbar_wait(dq_full, d_phase & 1);
        ++d_phase;
        tc_fence_after();
      }
#pragma unroll 1
      for (int c = 0; c < HS / 32; ++c) {
        uint32_t r[32];
        if (n > 0) {
          tmem_ld32(lane_base + 256 + c * 32, r);
          tmem_ld_wait(r);
        }
        if (!valid) continue;
        float4* dst = reinterpret_cast<float4*>(p.dq + row * HS + c * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4 v = n > 0 ? make_float4(__uint_as_float(r[4 * i]) * p.inv_scale,
                                         __uint_as_float(r[4 * i + 1]) * p.inv_scale,
                                         __uint_as_float(r[4 * i + 2]) * p.inv_scale,
                                         __uint_as_float(r[4 * i + 3]) * p.inv_scale)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
          if (p.accumulate) {
            const float4 a = dst[i];
            v.x += a.x;
            v.y += a.y;
            v.z += a.z;
            v.w += a.w;
          }
          dst[i] = v;
        }
      }
    }
  } else if (warp == C::kTmaWarp) {
    // ---------------------------------------------------- producer
    if (lane == 0) {
      uint32_t kv_it = 0, q_it = 0;
      for (uint32_t it = 0;; ++it) {
        const int u = atomicAdd(&p.sched[0], 1);
        mbar_wait(u_empty, (it & 1) ^ 1);
        *reinterpret_cast<volatile int*>(unit_slot) = u;
        mbar_arrive(u_full);
        if (u >= p.num_units) break;
        const uint32_t unit = p.units[u];
        const int qt = unit & 0xFFFF, h = (unit >> 16) & 0xFF, b = unit >> 24;
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
        for (int j = 0; j < n; ++j) {
          const int kt = p.tile_list[beg + j] & 0x7FFFFFFF;
          for (int which = 0; which < 2; ++which) {
            const uint32_t slot = kv_it % NS;
            mbar_wait(&kv_empty[slot], ((kv_it / NS) & 1) ^ 1);
            ++kv_it;
            mbar_arrive_expect_tx(&kv_full[slot], C::kTileBytes);
            const CUtensorMap* tm = which == 0 ? &p.tm_k : &p.tm_v;
            for (int sb = 0; sb < C::kSub; ++sb)
              tma_load_4d(sKV + slot * C::kTileBytes + sb * C::kSubBytes, tm, &kv_full[slot], sb * 64,
                          kvh, kt * 128, b);
          }
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
    const uint64_t q_desc = smem_desc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t do_desc = smem_desc_sw128(smem_u32(sDO), 16, 1024);
    const uint64_t kv_desc0 = smem_desc_sw128(smem_u32(sKV), 16, 1024);
    const uint64_t kvmn_desc0 = smem_desc_sw128(smem_u32(sKV), C::kSubBytes, 1024);
    uint32_t kv_it = 0, q_phase = 0, ds_phase = 0;
    auto ss = [&](uint32_t d, uint64_t ad, uint32_t slot) {  // D = A * B^T, B K-major from slot
      bwd_dispatch_slot<NS>(slot, [&](auto S) {
        constexpr int sl = decltype(S)::value;
        const uint64_t bd = kv_desc0 + static_cast<uint64_t>((sl * C::kTileBytes) >> 4);
        if (elect_one()) {
          if constexpr (HS == 128)
            mma_qk_hs128(d, ad, bd, C::kIdescSS, 0u);
          else
            mma_qk_hs64(d, ad, bd, C::kIdescSS, 0u);
        }
        __syncwarp();
      });
    };
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it, true);
      if (u >= p.num_units) break;
      const int qt = p.units[u] & 0xFFFF;
      const int n = p.tile_off[qt + 1] - p.tile_off[qt];
      if (n == 0) continue;
      mbar_wait(q_full, q_phase & 1);
      ++q_phase;
      tc_fence_after();
      for (int j = 0; j < n; ++j) {
        const uint32_t ki = kv_it + 2 * j, vi = ki + 1;
        mbar_wait(&kv_full[ki % NS], (ki / NS) & 1);
        mbar_wait(&kv_full[vi % NS], (vi / NS) & 1);
        tc_fence_after();
        ss(0, q_desc, ki % NS);     // S  = Q  K^T
        ss(128, do_desc, vi % NS);  // dP = dO V^T
        bwd_commit(s_full);
        if (j == n - 1) bwd_commit(q_empty);
        mbar_wait(ds_ready, ds_phase & 1);
        ++ds_phase;
        tc_fence_after();
        // dQ += dS K: K tile as the MN-major B operand
        bwd_dispatch_slot<NS>(ki % NS, [&](auto S) {
          constexpr int sl = decltype(S)::value;
          const uint64_t bd = kvmn_desc0 + static_cast<uint64_t>((sl * C::kTileBytes) >> 4);
          if (elect_one()) mma_pv_chain(256, 0, bd, C::kIdescTS, j > 0 ? 1u : 0u);
          __syncwarp();
        });
        bwd_commit(&kv_empty[ki % NS]);
        bwd_commit(&kv_empty[vi % NS]);
      }
      bwd_commit(dq_full);
      kv_it += 2 * n;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, 512);
}

// ============================================================ dk/dv kernel
// TMEM: S^T [0,128) (P^T bf16 over its first 64 columns), dP^T [128,256)
// (dS^T bf16 over its first 64), dV [256, 256+HS), dK [256+HS, 256+2HS).
// Q / dO tiles stream through the slot ring; K, V stay resident per unit.
template <int HS>
__global__ void __launch_bounds__(BwdCfg<HS>::kThreads, 1) fa_bwd_dkdv_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdCfg<HS>;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + C::kTileBytes;
  uint8_t* sQD = smem + 2 * C::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sQD + NS * C::kTileBytes);
  uint64_t* kv_full = bars;         // K + V landed
  uint64_t* kv_empty = bars + 1;
  uint64_t* s_full = bars + 2;      // S^T and dP^T in TMEM
  uint64_t* pd_ready = bars + 3;    // P^T, dS^T written (128 arrivals)
  uint64_t* acc_full = bars + 4;    // unit's last dV/dK MMA done
  uint64_t* qd_full = bars + 5;     // [NS]
  uint64_t* qd_empty = qd_full + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qd_empty + NS);
  int* unit_slot = reinterpret_cast<int*>(tmem_slot + 2);
  uint64_t* u_full = reinterpret_cast<uint64_t*>(unit_slot + 2);
  uint64_t* u_empty = u_full + 1;
  float* vec = reinterpret_cast<float*>(u_empty + 1);  // [2 parity][lse2 128 | delta 128 | qpos 128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(pd_ready, 128);
    mbar_init(acc_full, 1);
    mbar_init(u_full, 1);
    mbar_init(u_empty, 5);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&qd_full[s], 1);
      mbar_init(&qd_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == C::kMmaWarp) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tmem != 0) __trap();
  const int group = p.heads / p.kv_heads;

  auto get_unit = [&](uint32_t it, bool whole_warp) {
    mbar_wait(u_full, it & 1);
    const int u = *reinterpret_cast<volatile int*>(unit_slot);
    if (whole_warp) {
      __syncwarp();
      if (lane == 0) mbar_arrive(u_empty);
    } else {
      mbar_arrive(u_empty);
    }
    return u;
  };

  if (warp < 4) {
    // ---------------------------------------------------- compute warps (thread = key row)
    const int key_in_tile = warp * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const float sl2 = p.scale_log2;
    uint32_t s_phase = 0, a_phase = 0, vpar = 0;
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it, true);
      if (u >= p.num_units) break;
      const uint32_t unit = p.units[u];
      const int kt = unit & 0xFFFF, kvh = (unit >> 16) & 0xFF, b = unit >> 24;
      const int beg = p.tile_off[kt], n = p.tile_off[kt + 1] - beg;
      const int k_row = kt * 128 + key_in_tile;
      const int kpos = p.k_pos[k_row];
      for (int g = 0; g < group; ++g) {
        const int h = kvh * group + g;
        for (int j = 0; j < n; ++j) {
          const int entry = p.tile_list[beg + j];
          const int qt = entry & 0x7FFFFFFF;
          // this q tile's lse2 / delta / q positions -> shared (parity buffer)
          float* vb = vec + (vpar & 1) * 384;
          ++vpar;
          {
            const int qr = qt * 128 + key_in_tile;
            const bool ok = qr < p.q_len;
            const size_t r = (static_cast<size_t>(b) * p.q_len + (ok ? qr : 0)) * p.heads + h;
            vb[key_in_tile] = ok ? p.lse[r] * 1.4426950408889634f : INFINITY;  // padding rows: p = 0
            vb[128 + key_in_tile] = ok ? p.delta[r] : 0.f;
            vb[256 + key_in_tile] = __int_as_float(p.q_pos[qr]);
          }
          bwd_bar_sync(1, 128);
          mbar_wait(s_full, s_phase & 1);
          ++s_phase;
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t s[32], dp[32];
            tmem_ld32(lane_base + c * 32, s);
            tmem_ld32(lane_base + 128 + c * 32, dp);
            tmem_ld_wait(s);
            tmem_ld_wait(dp);
            uint32_t pp[16], pd[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int q0 = c * 32 + 2 * i, q1 = q0 + 1;
              float p0 = ex2(fmaf(__uint_as_float(s[2 * i]), sl2, -vb[q0]));
              float p1 = ex2(fmaf(__uint_as_float(s[2 * i + 1]), sl2, -vb[q1]));
              if (entry < 0) {
                if (kpos > __float_as_int(vb[256 + q0])) p0 = 0.f;
                if (kpos > __float_as_int(vb[256 + q1])) p1 = 0.f;
              }
              const float d0 = p0 * (__uint_as_float(dp[2 * i]) - vb[128 + q0]);
              const float d1 = p1 * (__uint_as_float(dp[2 * i + 1]) - vb[128 + q1]);
              pp[i] = pack_bf16x2(p0, p1);
              pd[i] = pack_bf16x2(d0, d1);
            }
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
                "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(lane_base + c * 16),
                "r"(pp[0]), "r"(pp[1]), "r"(pp[2]), "r"(pp[3]), "r"(pp[4]), "r"(pp[5]), "r"(pp[6]),
                "r"(pp[7]), "r"(pp[8]), "r"(pp[9]), "r"(pp[10]), "r"(pp[11]), "r"(pp[12]),
                "r"(pp[13]), "r"(pp[14]), "r"(pp[15])
                : "memory");
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
                "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(lane_base + 128 +
                                                                                     c * 16),
                "r"(pd[0]), "r"(pd[1]), "r"(pd[2]), "r"(pd[3]), "r"(pd[4]), "r"(pd[5]), "r"(pd[6]),
                "r"(pd[7]), "r"(pd[8]), "r"(pd[9]), "r"(pd[10]), "r"(pd[11]), "r"(pd[12]),
                "r"(pd[13]), "r"(pd[14]), "r"(pd[15])
                : "memory");
          }
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(pd_ready);
        }
      }
      // epilogue: dk (+)= dK / sqrt(hs), dv (+)= dV
      const bool any = n > 0;
      if (any) {
        mbar_wait(acc_full, a_phase & 1);
        ++a_phase;
        tc_fence_after();
      }
      const bool valid = k_row < p.k_len;
      const size_t krow = (static_cast<size_t>(b) * p.k_len + (valid ? k_row : 0)) * p.kv_heads + kvh;
#pragma unroll 1
      for (int which = 0; which < 2; ++which) {
        float* out = which == 0 ? p.dv : p.dk;
        const float sc = which == 0 ? 1.f : p.inv_scale;
        const uint32_t col = which == 0 ? 256 : 256 + HS;
#pragma unroll 1
        for (int c = 0; c < HS / 32; ++c) {
          uint32_t r[32];
          if (any) {
            tmem_ld32(lane_base + col + c * 32, r);
            tmem_ld_wait(r);
          }
          if (!valid) continue;
          float4* dst = reinterpret_cast<float4*>(out + krow * HS + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 v = any ? make_float4(__uint_as_float(r[4 * i]) * sc, __uint_as_float(r[4 * i + 1]) * sc,
                                         __uint_as_float(r[4 * i + 2]) * sc, __uint_as_float(r[4 * i + 3]) * sc)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            if (p.accumulate) {
              const float4 a = dst[i];
              v.x += a.x;
              v.y += a.y;
              v.z += a.z;
              v.w += a.w;
            }
            dst[i] = v;
          }
        }
      }
    }
  } else if (warp == C::kTmaWarp) {
    // ---------------------------------------------------- producer
    if (lane == 0) {
      uint32_t qd_it = 0, kv_it = 0;
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
        for (int g = 0; g < group; ++g) {
          const int h = kvh * group + g;
          for (int j = 0; j < n; ++j) {
            const int qt = p.tile_list[beg + j] & 0x7FFFFFFF;
            for (int which = 0; which < 2; ++which) {
              const uint32_t slot = qd_it % NS;
              mbar_wait(&qd_empty[slot], ((qd_it / NS) & 1) ^ 1);
              ++qd_it;
              mbar_arrive_expect_tx(&qd_full[slot], C::kTileBytes);
              const CUtensorMap* tm = which == 0 ? &p.tm_q : &p.tm_do;
              for (int sb = 0; sb < C::kSub; ++sb)
                tma_load_4d(sQD + slot * C::kTileBytes + sb * C::kSubBytes, tm, &qd_full[slot], sb * 64, h,
                            qt * 128, b);
            }
          }
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
    const uint64_t qd_desc0 = smem_desc_sw128(smem_u32(sQD), 16, 1024);
    const uint64_t qdmn_desc0 = smem_desc_sw128(smem_u32(sQD), C::kSubBytes, 1024);
    uint32_t qd_it = 0, kv_phase = 0, pd_phase = 0;
    for (uint32_t it = 0;; ++it) {
      const int u = get_unit(it, true);
      if (u >= p.num_units) break;
      const int kt = p.units[u] & 0xFFFF;
      const int n = p.tile_off[kt + 1] - p.tile_off[kt];
      if (n == 0) continue;
      mbar_wait(kv_full, kv_phase & 1);
      ++kv_phase;
      tc_fence_after();
      const int total = group * n;
      for (int i = 0; i < total; ++i) {
        const uint32_t qi = qd_it + 2 * i, di = qi + 1;
        mbar_wait(&qd_full[qi % NS], (qi / NS) & 1);
        mbar_wait(&qd_full[di % NS], (di / NS) & 1);
        tc_fence_after();
        bwd_dispatch_slot<NS>(qi % NS, [&](auto S) {  // S^T = K Q^T
          constexpr int sl = decltype(S)::value;
          const uint64_t bd = qd_desc0 + static_cast<uint64_t>((sl * C::kTileBytes) >> 4);
          if (elect_one()) {
            if constexpr (HS == 128)
              mma_qk_hs128(0, k_desc, bd, C::kIdescSS, 0u);
            else
              mma_qk_hs64(0, k_desc, bd, C::kIdescSS, 0u);
          }
          __syncwarp();
        });
        bwd_dispatch_slot<NS>(di % NS, [&](auto S) {  // dP^T = V dO^T
          constexpr int sl = decltype(S)::value;
          const uint64_t bd = qd_desc0 + static_cast<uint64_t>((sl * C::kTileBytes) >> 4);
          if (elect_one()) {
            if constexpr (HS == 128)
              mma_qk_hs128(128, v_desc, bd, C::kIdescSS, 0u);
            else
              mma_qk_hs64(128, v_desc, bd, C::kIdescSS, 0u);
          }
          __syncwarp();
        });
        bwd_commit(s_full);
        mbar_wait(pd_ready, pd_phase & 1);
        ++pd_phase;
        tc_fence_after();
        const uint32_t acc = i > 0 ? 1u : 0u;
        bwd_dispatch_slot<NS>(di % NS, [&](auto S) {  // dV += P^T dO
          constexpr int sl = decltype(S)::value;
          const uint64_t bd = qdmn_desc0 + static_cast<uint64_t>((sl * C::kTileBytes) >> 4);
          if (elect_one()) mma_pv_chain(256, 0, bd, C::kIdescTS, acc);
          __syncwarp();
        });
        bwd_dispatch_slot<NS>(qi % NS, [&](auto S) {  // dK += dS^T Q
          constexpr int sl = decltype(S)::value;
          const uint64_t bd = qdmn_desc0 + static_cast<uint64_t>((sl * C::kTileBytes) >> 4);
          if (elect_one()) mma_pv_chain(256 + HS, 128, bd, C::kIdescTS, acc);
          __syncwarp();
        });
        bwd_commit(&qd_empty[qi % NS]);
        bwd_commit(&qd_empty[di % NS]);
      }
      bwd_commit(acc_full);
      bwd_commit(kv_empty);
      qd_it += 2 * total;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kMmaWarp) tmem_dealloc(tmem, 512);
}

// ============================================================ small kernels
__global__ void delta_kernel(const uint16_t* o, const uint16_t* dout, float* delta,
                             int64_t rows, int hs) {
  // one warp per row: 16-byte loads, fp32 dot, shuffle reduction
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const uint16_t* a = o + row * hs;
  const uint16_t* bq = dout + row * hs;
  float acc = 0.f;
  for (int e = lane * 2; e < hs; e += 64) {
    const uint32_t x = *reinterpret_cast<const uint32_t*>(a + e);
    const uint32_t y = *reinterpret_cast<const uint32_t*>(bq + e);
    acc = fmaf(__uint_as_float(x << 16), __uint_as_float(y << 16), acc);
    acc = fmaf(__uint_as_float(x & 0xFFFF0000u), __uint_as_float(y & 0xFFFF0000u), acc);
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) delta[row] = acc;
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

template <class K>
cudaError_t set_smem(K kern, int bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace

cudaError_t launch_bwd_dq(const BwdParams& p, int hs, int grid, cudaStream_t stream) {
  if (hs == 128) {
    static cudaError_t once = set_smem(fa_bwd_dq_kernel<128>, BwdCfg<128>::kSmemBytes);
    if (once != cudaSuccess) return once;
    fa_bwd_dq_kernel<128><<<grid, BwdCfg<128>::kThreads, BwdCfg<128>::kSmemBytes, stream>>>(p);
  } else if (hs == 64) {
    static cudaError_t once = set_smem(fa_bwd_dq_kernel<64>, BwdCfg<64>::kSmemBytes);
    if (once != cudaSuccess) return once;
    fa_bwd_dq_kernel<64><<<grid, BwdCfg<64>::kThreads, BwdCfg<64>::kSmemBytes, stream>>>(p);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_bwd_dkdv(const BwdParams& p, int hs, int grid, cudaStream_t stream) {
  if (hs == 128) {
    static cudaError_t once = set_smem(fa_bwd_dkdv_kernel<128>, BwdCfg<128>::kSmemBytes);
    if (once != cudaSuccess) return once;
    fa_bwd_dkdv_kernel<128><<<grid, BwdCfg<128>::kThreads, BwdCfg<128>::kSmemBytes, stream>>>(p);
  } else if (hs == 64) {
    static cudaError_t once = set_smem(fa_bwd_dkdv_kernel<64>, BwdCfg<64>::kSmemBytes);
    if (once != cudaSuccess) return once;
    fa_bwd_dkdv_kernel<64><<<grid, BwdCfg<64>::kThreads, BwdCfg<64>::kSmemBytes, stream>>>(p);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_bwd_delta(const void* o, const void* dout, float* delta, int64_t rows, int hs,
                             cudaStream_t stream) {
  if (rows == 0) return cudaSuccess;
  const int64_t threads = rows * 32;
  const int grid = static_cast<int>((threads + 255) / 256);
  delta_kernel<<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(o),
                                         static_cast<const uint16_t*>(dout), delta, rows, hs);
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
