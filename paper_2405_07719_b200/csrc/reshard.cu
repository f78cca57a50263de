// reshard.cu — the Ulysses pack/unpack transposes (and head-size padding).
//
// Restates the data movement of scatter_heads_gather_seq /
// scatter_seq_gather_heads (reference src/usp/all_to_all_4d.cpp:27-39,
// 42-57, 75-87, 90-105) as one HBM-bound row-permutation kernel: every
// destination row (one head_size vector) is fetched from an affine source
// row index over four loop dimensions. 16-byte vectors, one thread per
// vector, grid sized in waves of the SM count; head sizes that are not a
// multiple of 8 take the scalar path (only small test shapes do).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "reshard.hpp"

namespace uspb200 {

template <int VEC>
__global__ void __launch_bounds__(256) row_permute_kernel(RowPermute p) {
  const int64_t chunks = (p.hs_dst + VEC - 1) / VEC;
  const int64_t total = p.dims[0] * p.dims[1] * p.dims[2] * p.dims[3] * chunks;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = idx % chunks;
    int64_t r = idx / chunks;
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
    const int64_t e = c * VEC;
    if (VEC == 8 && e + 8 <= p.hs_src) {
      *reinterpret_cast<uint4*>(dst + e) = __ldg(reinterpret_cast<const uint4*>(src + e));
    } else {
      for (int v = 0; v < VEC && e + v < p.hs_dst; ++v)
        dst[e + v] = (e + v < p.hs_src) ? src[e + v] : __float2bfloat16(0.f);
    }
  }
}

cudaError_t launch_row_permute(const RowPermute& p, int num_sms, cudaStream_t stream) {
  const bool vec = (p.hs_src % 8 == 0) && (p.hs_dst % 8 == 0) &&
                   (reinterpret_cast<uintptr_t>(p.src) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(p.dst) % 16 == 0);
  const int v = vec ? 8 : 1;
  const int64_t chunks = (p.hs_dst + v - 1) / v;
  const int64_t total = p.dims[0] * p.dims[1] * p.dims[2] * p.dims[3] * chunks;
  if (total == 0) return cudaSuccess;
  const int64_t blocks_needed = (total + 255) / 256;
  const int64_t cap = int64_t(num_sms) * 8;  // 8 resident 256-thread CTAs per SM
  const int grid = static_cast<int>(blocks_needed < cap ? blocks_needed : cap);
  if (vec)
    row_permute_kernel<8><<<grid, 256, 0, stream>>>(p);
  else
    row_permute_kernel<1><<<grid, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace uspb200
