// fa_fwd.hpp — host/device contract of the per-block attention kernel.
//
// One launch folds one K/V block (one ring step) into the attention state
// of every (batch, q-head, 128-row query tile) of this rank:
//   SoftmaxState::update  (reference src/numerics/attention.cpp:181-230)
//   finalize + logsumexp  (attention.cpp:232-264)
//   ring-step LSE merge   (the online-softmax fold across the R steps of
//                          src/usp/ring_attention.cpp:62-75)
// The causal mask is the reference BlockMask::causal (attention.hpp:32-34):
// key j is hidden from query i iff k_pos[j] > q_pos[i]. Tile classification
// (full / partial / skipped) is done on the host by plan.cpp.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace uspb200 {

constexpr int kTileM = 128;  // query rows per tile (TMEM lanes)
constexpr int kTileN = 128;  // keys per K/V tile
constexpr int kTraceTiles = 256;
constexpr int kTraceEvents = 16;

enum class EpiMode : int {
  kSingle = 0,  // only step: write bf16 O + natural-log LSE
  kFirst = 1,   // first of several steps: write fp32 (O, lse2) running state
  kMiddle = 2,  // merge into the running state
  kLast = 3,    // merge, then write bf16 O + natural-log LSE
};

struct FwdParams {
  CUtensorMap tm_q;  // (hs, heads, q_len, batch) bf16, box (64, 1, 128, 1), SW128
  CUtensorMap tm_k;  // (hs, kv_heads, k_len, batch)
  CUtensorMap tm_v;
  CUtensorMap tm_k64;  // K with 64-row boxes (2SM cluster mode: each CTA loads 64 keys)

  void* o;            // bf16 (batch, q_len, heads, hs)  [kSingle, kLast]
  float* lse;         // fp32 (batch, q_len, heads), natural log [kSingle, kLast]
  float* o_acc;       // fp32 running O (batch, q_len, heads, hs) [kFirst..kLast]
  float* lse_acc;     // fp32 running LSE, log2 domain           [kFirst..kLast]

  const uint32_t* units;     // packed work units: q_tile | hp << 16 | b << 24 (pair_rows:
                             // tile pair | head << 16 | b << 24)
  const int32_t* tile_off;   // CSR row offsets per q tile (n_q_tiles + 1)
  const int32_t* tile_list;  // k tile index | partial << 31
  const int32_t* q_pos;      // effective query positions, padded to 128
  const int32_t* k_pos;      // effective key positions, padded to 128 (INT_MAX)

  int* sched;  // [0] next-unit ticket, [1] finished-CTA count; zero between launches
  int num_units;
  int batch, q_len, k_len, heads, kv_heads;
  int mode;          // EpiMode
  // Direct O (Ulysses out fused into the epilogue): when o_peer[0] != null,
  // bf16 O row r of this rank's head-sharded block goes to Ulysses member
  // p = r / o_part_rows, straight into that member's receive buffer at
  // [o_me][r - p*o_part_rows][head][hs] (peer memory over NVLink).
  void* o_peer[16];
  int o_part_rows;   // T: rows per Ulysses part
  int o_me;          // this rank's index in its Ulysses group
  int cluster;       // 1/2: 2-CTA clusters (TMA multicast / cta_group::2 MMAs), unit hp = head quad
  int pair_rows;     // 1: a unit is two adjacent 128-row tiles of one head
                     //    (q_tile field = tile pair); 0: two heads of a pair
  float scale_log2;  // log2(e) / sqrt(head_size)
  int kv_hint;       // L2 policy for K/V tile loads: 0 normal, 1 evict_last
  // Development tracing (nullptr in production): clock64 stamps of CTA 0's
  // first kTraceTiles tiles, [event][tile]; see tools/trace_fa.py.
  unsigned long long* trace;
  int debug_flags;  // development: bit 0 = skip the softmax math (pipeline-only timing)
  // Parity instrumentation (nullptr in production): +1 per (warp, key tile)
  // whose lazy O rescale fired (running max grew by > 8 in log2 units), so
  // the tests can prove the alpha != 1 branch ran (usp_engine_debug_counters).
  unsigned long long* rescale_count;
};

// cudaFuncSetAttribute is per device: opt a kernel in to its dynamic shared
// memory once on every device it is launched on (`done`: one bit per device).
template <class K>
inline cudaError_t ensure_smem_attr(K kern, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

}  // namespace uspb200
