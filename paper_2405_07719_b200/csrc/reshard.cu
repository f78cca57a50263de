// reshard.cu — the Ulysses pack/unpack transposes (and head-size padding).
//
// Restates the data movement of scatter_heads_gather_seq /
// scatter_seq_gather_heads (reference src/usp/all_to_all_4d.cpp:27-39,
// 42-57, 75-87, 90-105) as one HBM-bound row-permutation kernel: every
// destination row (one head_size vector) is fetched from an affine source
// row index over four loop dimensions.
//
// Fast path (every shape the engine moves: 16-byte aligned rows, fewer than
// 2^31 vectors): 32-bit index arithmetic, and each thread keeps kUnroll
// independent 16-byte loads in flight before storing them — the first
// version (64-bit div/mod per vector, one load in flight) reached 3.3 TB/s;
// HBM-bound work should run near the copy bandwidth. Head sizes that are not
// a multiple of 8 (or padding to a larger destination row) take the scalar
// path (small test shapes only).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "reshard.hpp"

namespace uspb200 {

namespace {

constexpr int kUnroll = 4;

struct Dims32 {
  uint32_t d1, d2, d3, chunks;  // loop extents (d0 implied by total)
  uint32_t s0, s1, s2, s3;      // source row strides
  uint32_t t0, t1, t2, t3;      // destination row strides
};

__device__ __forceinline__ void locate(const Dims32& d, uint32_t idx, uint32_t& srow, uint32_t& drow,
                                       uint32_t& c) {
  c = idx % d.chunks;
  uint32_t r = idx / d.chunks;
  const uint32_t i3 = r % d.d3;
  r /= d.d3;
  const uint32_t i2 = r % d.d2;
  r /= d.d2;
  const uint32_t i1 = r % d.d1;
  const uint32_t i0 = r / d.d1;
  srow = i0 * d.s0 + i1 * d.s1 + i2 * d.s2 + i3 * d.s3;
  drow = i0 * d.t0 + i1 * d.t1 + i2 * d.t2 + i3 * d.t3;
}

// 16-byte vectors, hs_src == hs_dst == 8 * chunks, all indices < 2^31.
__global__ void __launch_bounds__(256) row_permute_vec(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                       Dims32 d, uint32_t total) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < total; base += stride * kUnroll) {
    uint4 v[kUnroll];
    uint32_t out[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t idx = base + u * stride;
      if (idx < total) {
        uint32_t srow, drow, c;
        locate(d, idx, srow, drow, c);
        v[u] = __ldg(src + srow * d.chunks + c);
        out[u] = drow * d.chunks + c;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (base + u * stride < total) dst[out[u]] = v[u];
  }
}

// General path: any head sizes (zero padding / truncation), 64-bit indices.
__global__ void __launch_bounds__(256) row_permute_scalar(RowPermute p) {
  const int64_t total = p.dims[0] * p.dims[1] * p.dims[2] * p.dims[3] * p.hs_dst;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = idx % p.hs_dst;
    int64_t r = idx / p.hs_dst;
    const int64_t i3 = r % p.dims[3];
    r /= p.dims[3];
    const int64_t i2 = r % p.dims[2];
    r /= p.dims[2];
    const int64_t i1 = r % p.dims[1];
    const int64_t i0 = r / p.dims[1];
    const int64_t srow = i0 * p.src_stride[0] + i1 * p.src_stride[1] + i2 * p.src_stride[2] +
                         i3 * p.src_stride[3];
    const int64_t drow = i0 * p.dst_stride[0] + i1 * p.dst_stride[1] + i2 * p.dst_stride[2] +
                         i3 * p.dst_stride[3];
    const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(p.src) + srow * p.hs_src;
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.dst) + drow * p.hs_dst;
    dst[e] = e < p.hs_src ? src[e] : __float2bfloat16(0.f);
  }
}

int64_t max_row(const RowPermute& p, const int64_t* stride) {
  int64_t m = 0;
  for (int i = 0; i < 4; ++i) m += (p.dims[i] - 1) * stride[i];
  return m;
}

}  // namespace

cudaError_t launch_row_permute(const RowPermute& p, int num_sms, cudaStream_t stream) {
  const int64_t rows = p.dims[0] * p.dims[1] * p.dims[2] * p.dims[3];
  if (rows == 0 || p.hs_dst == 0) return cudaSuccess;
  const int64_t chunks = p.hs_dst / 8;
  const int64_t total_vec = rows * chunks;
  const bool vec = p.hs_src == p.hs_dst && p.hs_dst % 8 == 0 &&
                   reinterpret_cast<uintptr_t>(p.src) % 16 == 0 && reinterpret_cast<uintptr_t>(p.dst) % 16 == 0 &&
                   total_vec < (int64_t(1) << 31) && (max_row(p, p.src_stride) + 1) * chunks < (int64_t(1) << 31) &&
                   (max_row(p, p.dst_stride) + 1) * chunks < (int64_t(1) << 31);
  const int64_t cap = int64_t(num_sms) * 8;  // 8 resident 256-thread CTAs per SM
  if (vec) {
    Dims32 d{uint32_t(p.dims[1]), uint32_t(p.dims[2]), uint32_t(p.dims[3]), uint32_t(chunks),
             uint32_t(p.src_stride[0]), uint32_t(p.src_stride[1]), uint32_t(p.src_stride[2]), uint32_t(p.src_stride[3]),
             uint32_t(p.dst_stride[0]), uint32_t(p.dst_stride[1]), uint32_t(p.dst_stride[2]), uint32_t(p.dst_stride[3])};
    const int64_t blocks = (total_vec + 256 * kUnroll - 1) / (256 * kUnroll);
    const int grid = static_cast<int>(blocks < cap ? blocks : cap);
    row_permute_vec<<<grid, 256, 0, stream>>>(static_cast<const uint4*>(p.src), static_cast<uint4*>(p.dst), d,
                                              uint32_t(total_vec));
  } else {
    const int64_t total = rows * p.hs_dst;
    const int64_t blocks = (total + 255) / 256;
    const int grid = static_cast<int>(blocks < cap ? blocks : cap);
    row_permute_scalar<<<grid, 256, 0, stream>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace uspb200
