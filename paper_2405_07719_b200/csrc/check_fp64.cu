// check_fp64.cu — the `simulate` command's single-device fp64 check, on the GPU.
//
// The reference's simulate (src/api/commands.cpp:139-158) compares the
// distributed result against reference_attention / reference_attention_grad
// (src/numerics/attention.cpp:51-170) run in fp64 on the same inputs. This is
// the same computation as plain fp64 CUDA (one warp per row, lanes split the
// head dimension, the reference's two-pass max / exp-sum per row), so a
// `"check": true` request never leaves the device for its arithmetic:
//   O_i   = sum_j exp(s_ij - m_i) v_j / l_i,   s_ij = q_i.k_j / sqrt(hs)
//   dP_ij = dO_i . v_j,  pdp_i = sum_j p_ij dP_ij,  dS_ij = p_ij (dP_ij - pdp_i)
//   dQ_i  = sum_j dS_ij k_j / sqrt(hs);  dK_j = sum_i dS_ij q_i / sqrt(hs);
//   dV_j  = sum_i p_ij dO_i
// over global positions (key j visible to query i iff j <= i when causal),
// GQA head h reading kv head h / (hc / kv). Bandwidth/latency-bound fp64; it
// is a correctness check, not a hot path.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

namespace uspb200 {
namespace {

constexpr int kMaxPerLane = 4;  // hs <= 128

struct RefDims {
  int64_t batch, seq;
  int heads, kv_heads, hs;
  int causal;
  double inv_scale;
};

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ double dot_row(const double* a, const double* b, int hs, int lane) {
  double s = 0;
  for (int d = lane; d < hs; d += 32) s += a[d] * b[d];
  return warp_sum(s);
}

// One warp per (b, i, h): m_i, l_i (softmax statistics) and O_i.
__global__ void ref_fwd_rows(RefDims d, const double* q, const double* k, const double* v, double* out,
                             double* row_m, double* row_l) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= d.batch * d.seq * d.heads) return;
  const int h = int(row % d.heads);
  const int64_t i = (row / d.heads) % d.seq, b = row / (int64_t(d.heads) * d.seq);
  const int kvh = h / (d.heads / d.kv_heads);
  const double* qr = q + row * d.hs;
  const int64_t jmax = d.causal ? i : d.seq - 1;
  double m = -INFINITY;
  for (int64_t j = 0; j <= jmax; ++j)
    m = fmax(m, dot_row(qr, k + ((b * d.seq + j) * d.kv_heads + kvh) * d.hs, d.hs, lane) * d.inv_scale);
  double l = 0, acc[kMaxPerLane] = {0, 0, 0, 0};
  for (int64_t j = 0; j <= jmax; ++j) {
    const int64_t kr = ((b * d.seq + j) * d.kv_heads + kvh) * d.hs;
    const double w = exp(dot_row(qr, k + kr, d.hs, lane) * d.inv_scale - m);
    l += w;
#pragma unroll
    for (int c = 0; c < kMaxPerLane; ++c)
      if (lane + 32 * c < d.hs) acc[c] += w * v[kr + lane + 32 * c];
  }
#pragma unroll
  for (int c = 0; c < kMaxPerLane; ++c)
    if (lane + 32 * c < d.hs) out[row * d.hs + lane + 32 * c] = acc[c] / l;
  if (lane == 0) {
    row_m[row] = m;
    row_l[row] = l;
  }
}

// One warp per (b, i, h): pdp_i and dQ_i.
__global__ void ref_dq_rows(RefDims d, const double* q, const double* k, const double* v, const double* dout,
                            const double* row_m, const double* row_l, double* pdp_out, double* dq) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= d.batch * d.seq * d.heads) return;
  const int h = int(row % d.heads);
  const int64_t i = (row / d.heads) % d.seq, b = row / (int64_t(d.heads) * d.seq);
  const int kvh = h / (d.heads / d.kv_heads);
  const double* qr = q + row * d.hs;
  const double* dor = dout + row * d.hs;
  const int64_t jmax = d.causal ? i : d.seq - 1;
  const double m = row_m[row], l = row_l[row];
  double pdp = 0;
  for (int64_t j = 0; j <= jmax; ++j) {
    const int64_t kr = ((b * d.seq + j) * d.kv_heads + kvh) * d.hs;
    const double p = exp(dot_row(qr, k + kr, d.hs, lane) * d.inv_scale - m) / l;
    pdp += p * dot_row(dor, v + kr, d.hs, lane);
  }
  double acc[kMaxPerLane] = {0, 0, 0, 0};
  for (int64_t j = 0; j <= jmax; ++j) {
    const int64_t kr = ((b * d.seq + j) * d.kv_heads + kvh) * d.hs;
    const double p = exp(dot_row(qr, k + kr, d.hs, lane) * d.inv_scale - m) / l;
    const double ds = p * (dot_row(dor, v + kr, d.hs, lane) - pdp) * d.inv_scale;
#pragma unroll
    for (int c = 0; c < kMaxPerLane; ++c)
      if (lane + 32 * c < d.hs) acc[c] += ds * k[kr + lane + 32 * c];
  }
#pragma unroll
  for (int c = 0; c < kMaxPerLane; ++c)
    if (lane + 32 * c < d.hs) dq[row * d.hs + lane + 32 * c] = acc[c];
  if (lane == 0) pdp_out[row] = pdp;
}

// One warp per (b, j, kv head): dK_j and dV_j over the GQA group's q heads.
__global__ void ref_dkdv_rows(RefDims d, const double* q, const double* k, const double* v, const double* dout,
                              const double* row_m, const double* row_l, const double* pdp, double* dk,
                              double* dv) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= d.batch * d.seq * d.kv_heads) return;
  const int kvh = int(row % d.kv_heads);
  const int64_t j = (row / d.kv_heads) % d.seq, b = row / (int64_t(d.kv_heads) * d.seq);
  const int group = d.heads / d.kv_heads;
  const double* kr = k + row * d.hs;
  const double* vr = v + row * d.hs;
  double ak[kMaxPerLane] = {0, 0, 0, 0}, av[kMaxPerLane] = {0, 0, 0, 0};
  for (int g = 0; g < group; ++g) {
    const int h = kvh * group + g;
    for (int64_t i = d.causal ? j : 0; i < d.seq; ++i) {
      const int64_t qrow = (b * d.seq + i) * d.heads + h;
      const double* qr = q + qrow * d.hs;
      const double* dor = dout + qrow * d.hs;
      const double p = exp(dot_row(qr, kr, d.hs, lane) * d.inv_scale - row_m[qrow]) / row_l[qrow];
      const double ds = p * (dot_row(dor, vr, d.hs, lane) - pdp[qrow]) * d.inv_scale;
#pragma unroll
      for (int c = 0; c < kMaxPerLane; ++c) {
        if (lane + 32 * c < d.hs) {
          ak[c] += ds * qr[lane + 32 * c];
          av[c] += p * dor[lane + 32 * c];
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kMaxPerLane; ++c) {
    if (lane + 32 * c < d.hs) {
      dk[row * d.hs + lane + 32 * c] = ak[c];
      dv[row * d.hs + lane + 32 * c] = av[c];
    }
  }
}

}  // namespace

// Device pointers, (batch, seq, heads|kv_heads, hs) row-major fp64.
// out/dq like q; dk/dv like k. scratch: 3 * batch * seq * heads doubles.
cudaError_t reference_attention_fp64(int64_t batch, int64_t seq, int heads, int kv_heads, int hs, bool causal,
                                     const double* q, const double* k, const double* v, const double* dout,
                                     double* out, double* dq, double* dk, double* dv, double* scratch,
                                     cudaStream_t st) {
  if (hs > 32 * kMaxPerLane) return cudaErrorInvalidValue;
  RefDims d{batch, seq, heads, kv_heads, hs, causal ? 1 : 0, 1.0 / std::sqrt(double(hs))};
  const int64_t rows = batch * seq * heads, kvrows = batch * seq * kv_heads;
  double* m = scratch;
  double* l = scratch + rows;
  double* pdp = scratch + 2 * rows;
  const int threads = 256, per_block = threads / 32;
  ref_fwd_rows<<<unsigned((rows + per_block - 1) / per_block), threads, 0, st>>>(d, q, k, v, out, m, l);
  if (dout) {
    ref_dq_rows<<<unsigned((rows + per_block - 1) / per_block), threads, 0, st>>>(d, q, k, v, dout, m, l, pdp,
                                                                                  dq);
    ref_dkdv_rows<<<unsigned((kvrows + per_block - 1) / per_block), threads, 0, st>>>(d, q, k, v, dout, m, l,
                                                                                      pdp, dk, dv);
  }
  return cudaGetLastError();
}

}  // namespace uspb200
