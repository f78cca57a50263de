// reshard.hpp — row-permutation copy used for the Ulysses pack/unpack.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace uspb200 {

// dst_row(i0..i3) <- src_row(i0..i3), rows of bf16; strides in rows.
// Rows are hs_src / hs_dst elements long; extra destination elements are
// zero-filled, extra source elements dropped (exact head-size padding).
struct RowPermute {
  const void* src = nullptr;
  void* dst = nullptr;
  int64_t dims[4] = {1, 1, 1, 1};
  int64_t src_stride[4] = {0, 0, 0, 0};
  int64_t dst_stride[4] = {0, 0, 0, 0};
  int64_t hs_src = 0, hs_dst = 0;
};

cudaError_t launch_row_permute(const RowPermute& p, int num_sms, cudaStream_t stream);
// Several permutations, one launch of the TMA bulk-copy kernel when all of
// them are runs of contiguous rows (every engine pack / unpack at a native
// head size); *launches = kernels launched.
cudaError_t launch_row_permute_multi(const RowPermute* ps, int n, int num_sms, cudaStream_t stream,
                                     int* launches);

}  // namespace uspb200
