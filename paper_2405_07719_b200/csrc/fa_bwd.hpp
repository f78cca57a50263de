// fa_bwd.hpp — host/device contract of the attention backward kernels
// (SURVEY §8(f) #1). Restates the reference's per-block backward
// attention_block_backward (src/numerics/attention.cpp:282-324):
//   p  = exp(s - lse),           s = q.k / sqrt(hs)  (masked -> 0)
//   dp = dO . v,  ds = p (dp - delta) / sqrt(hs),  delta = rowsum(dO * O)
//   dQ += ds K,  dK += ds^T Q,  dV += p^T dO
// as two tcgen05 kernels (dQ per query tile; dK/dV per key tile, summed over
// the GQA group's query heads) accumulating in fp32.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace uspb200 {

struct BwdParams {
  CUtensorMap tm_q, tm_k, tm_v, tm_do;  // (hs, heads, len, batch) bf16, box (64,1,128,1), SW128
  // fused kernel: the fp32 dQ accumulator (hs, heads, q_len, batch), box
  // (32, 1, 32, 1), 128B swizzle — target of the TMA reductions
  CUtensorMap tm_dq;
  const float* lse;    // natural-log LSE (batch, q_len, heads)
  const float* delta;  // rowsum(dO * O) (batch, q_len, heads)
  float* dq;           // fp32 (batch, q_len, heads, hs)      [dq kernel]
  float* dk;           // fp32 (batch, k_len, kv_heads, hs)   [dkdv kernel]
  float* dv;

  const uint32_t* units;     // dq: q_tile | head << 16 | b << 24; dkdv: k_tile | kv_head << 16 | b << 24
  const int32_t* tile_off;   // CSR over the unit's tile dimension
  const int32_t* tile_list;  // other-dimension tile | partial << 31
  const int32_t* q_pos;      // effective positions (see StepPlan), padded to 128
  const int32_t* k_pos;
  int* sched;                // unit tickets, zero between launches
  // dK/dV kernel: per (batch, q head, 128-row q tile) the 3 x 128 floats
  // {-lse * log2(e) (-INF on padding rows), -delta, q position} laid out
  // contiguously ([b][h][q tile][3][128], filled by launch_bwd_delta) so the
  // TMA warp bulk-copies them next to the Q tile
  const float* qvec;
  int n_q_tiles;  // q tiles per (batch, head) in qvec
  int cluster;    // dq kernel: 1 = 2-CTA clusters over head pairs (unit head field = pair)

  int num_units;
  int batch, q_len, k_len, heads, kv_heads;
  float scale_log2;  // log2(e) / sqrt(head_size)
  float inv_scale;   // 1 / sqrt(head_size)
  int accumulate;    // 0: write the fp32 outputs, 1: add into them
  // development (USPB_TRACE builds, USP_BWD_TRACE=dq|dkdv): clock64 stamps of
  // CTA 0, [event][q tile] over the first kTraceTiles tiles; tools/trace_bwd.py
  unsigned long long* trace;
};

cudaError_t launch_bwd_dq(const BwdParams& p, int hs, int grid, cudaStream_t stream);
cudaError_t launch_bwd_dkdv(const BwdParams& p, int hs, int grid, cudaStream_t stream);
// Both in one kernel (kernel head size 64 or 128): units / CSR as for the dK/dV kernel
// (transpose_plan, single key tiles); dK / dV written like the dK/dV kernel,
// dQ (scaled) REDUCED into p.dq with fp32 atomics (caller zeroes it first).
cudaError_t launch_bwd_fused(const BwdParams& p, int hs, int grid, cudaStream_t stream);
// delta[row] = sum_s o[row][s] * dout[row][s]  (output_dot_rows, attention.cpp:266-280)
// over rows (b, t, h) of a (batch, q_len, heads, hs) tensor; with qvec also
// the dK/dV kernel's per-q-tile vectors (see BwdParams::qvec) from lse and
// the effective q positions (padded to whole tiles), the -delta entries
// multiplied by qvec_delta_scale (1 for the dK/dV kernel; 1/sqrt(hs) for the
// fused kernel, whose dS carries the softmax scale).
cudaError_t launch_bwd_delta(const void* o, const void* dout, float* delta, int64_t batch, int64_t q_len,
                             int heads, int hs, const float* lse, const int32_t* q_pos, float* qvec,
                             float qvec_delta_scale, cudaStream_t stream);
// acc = blk + acc, n fp32 elements (n % 4 == 0): the ring's circulating
// dK/dV partial plus this step's block (add_into, ring_attention.cpp:129-134).
cudaError_t launch_add_f32(const float* blk, float* acc, int64_t n, cudaStream_t stream);
// dst = bf16(src [+ src2]), rows of hs_src -> hs_dst (drops padding);
// the sum is (src + src2) in that order (ring_attention.cpp:145-150).
cudaError_t launch_cast_rows(const float* src, const float* src2, void* dst, int64_t rows, int hs_src,
                             int hs_dst, cudaStream_t stream);

}  // namespace uspb200
