// reshard.cu — the Ulysses pack/unpack transposes (and head-size padding).
//
// Restates the data movement of scatter_heads_gather_seq /
// scatter_seq_gather_heads (reference src/usp/all_to_all_4d.cpp:27-39,
// 42-57, 75-87, 90-105) as one HBM-bound row-permutation kernel: every
// destination row (one head_size vector) is fetched from an affine source
// row index over four loop dimensions.
//
// TMA path (every permutation the engine issues at a native head size):
// source and destination are two strided views of the same logical
// (i0, i1, i2, i3, element) space, so a permutation is a TMA tensor copy —
// each box (all hs elements x up to 256 i3 rows x b2 i2 rows) is loaded with
// cp.async.bulk.tensor from the source map and stored with
// cp.async.bulk.tensor to the destination map at the SAME coordinates; the
// strides in the two tensor maps do the transpose. One issuing lane per CTA
// keeps a ring of shared-memory boxes in flight; no per-element instructions,
// and ONE launch for several tensors (Q, K and V together; every peer part of
// the direct exchange). Vector path (fallback): 32-bit index arithmetic,
// 16-byte loads with kUnroll in flight per thread. Head sizes that are not a
// multiple of 8 (or padding to a larger destination row) take the scalar
// path (small test shapes only).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <cuda.h>

#include "ptx_sm100.cuh"
#include "plan.hpp"
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

// ------------------------------------------------------------------ TMA path
namespace {
constexpr int kTmaSlots = 6;
constexpr int kTmaAhead = 4;          // loads in flight ahead of the stores
constexpr int kTmaBoxBytes = 32768;
constexpr int kMaxTmaJobs = 48;

struct alignas(64) TmaJob {
  CUtensorMap src, dst;                // 5-D (hs, d3, d2, d1, d0) views
  int n3, n2, n1;                      // boxes along d3, d2, d1 (d0: the rest)
  int b3, b2;                          // box extent along d3, d2
  int bytes;                           // full-box bytes (TMA zero-fills / clips the edges)
  int first;                           // prefix of boxes over the jobs
  // map dims 2..4 <- logical outer coordinate (0: d2, 1: d1, 2: d0), per map:
  // each map orders its outer dims by stride (box-1 dims do not change the
  // box's shared-memory layout, so the two maps may order them differently)
  unsigned char ps[3], pd[3];
};
struct TmaParams {
  TmaJob job[kMaxTmaJobs];
  int njobs, total;
};

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2, int c3,
                                             int c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}

__device__ __forceinline__ void box_coords(const TmaParams& p, int i, const TmaJob*& j, int& c1, int& c2, int& c3,
                                           int& c4) {
  int k = 0;
  while (k + 1 < p.njobs && p.job[k + 1].first <= i) ++k;
  j = &p.job[k];
  int r = i - j->first;
  const int i3 = r % j->n3;
  r /= j->n3;
  const int i2 = r % j->n2;
  r /= j->n2;
  const int i1 = r % j->n1;
  c4 = r / j->n1;
  c1 = i3 * j->b3;
  c2 = i2 * j->b2;
  c3 = i1;
}

__global__ void __launch_bounds__(32, 1) reshard_tma_kernel(const __grid_constant__ TmaParams p) {
  extern __shared__ __align__(1024) uint8_t tma_smem[];
  __shared__ __align__(8) uint64_t bar[kTmaSlots];
  if (threadIdx.x != 0) return;  // one issuing lane
  for (int s = 0; s < kTmaSlots; ++s) ptx::mbar_init(&bar[s], 1);
  ptx::fence_barrier_init();
  const uint32_t base = (ptx::smem_u32(tma_smem) + 1023u) & ~1023u;
  const int cnt = p.total > int(blockIdx.x) ? (p.total - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x) : 0;
  for (int k = 0; k < cnt + kTmaAhead; ++k) {
    if (k < cnt) {  // load box k into slot k % S
      const int slot = k % kTmaSlots;
      // stores issued so far: boxes < k - A; the slot's previous box k - S
      // must have been read: at most S - A - 1 newer stores may be pending
      if (k >= kTmaSlots) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kTmaSlots - kTmaAhead - 1) : "memory");
      const TmaJob* j;
      int c1, c2, c3, c4;
      box_coords(p, int(blockIdx.x) + k * int(gridDim.x), j, c1, c2, c3, c4);
      ptx::mbar_arrive_expect_tx(&bar[slot], static_cast<uint32_t>(j->bytes));
      const int L[3] = {c2, c3, c4};
      tma_load_5d(base + slot * kTmaBoxBytes, &j->src, &bar[slot], 0, c1, L[j->ps[0]], L[j->ps[1]], L[j->ps[2]]);
    }
    if (k >= kTmaAhead && k - kTmaAhead < cnt) {  // store box k - A
      const int m = k - kTmaAhead;
      const int slot = m % kTmaSlots;
      ptx::mbar_wait(&bar[slot], static_cast<uint32_t>((m / kTmaSlots) & 1));
      const TmaJob* j;
      int c1, c2, c3, c4;
      box_coords(p, int(blockIdx.x) + m * int(gridDim.x), j, c1, c2, c3, c4);
      const int L[3] = {c2, c3, c4};
      tma_store_5d(&j->dst, base + slot * kTmaBoxBytes, 0, c1, L[j->pd[0]], L[j->pd[1]], L[j->pd[2]]);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// RowPermute -> TMA job; false when the shape does not fit the TMA path.
bool to_tma_job(const RowPermute& p, TmaJob& j) {
  const EncodeTiledFn enc = encode_tiled();
  if (!enc || p.hs_src != p.hs_dst || p.hs_src > 256 || (p.hs_src * 2) % 16) return false;
  if (p.src_stride[3] != 1 || p.dst_stride[3] != 1) return false;
  const int64_t row = p.hs_src * 2;
  for (int k = 0; k < 4; ++k)
    if (p.dims[k] < 1 || p.dims[k] > (int64_t(1) << 31)) return false;
  if (reinterpret_cast<uintptr_t>(p.src) % 16 || reinterpret_cast<uintptr_t>(p.dst) % 16) return false;
  const int b3 = static_cast<int>(std::min<int64_t>(p.dims[3], 256));
  const int64_t box_row_bytes = int64_t(b3) * row;
  if (box_row_bytes > kTmaBoxBytes) return false;
  const int b2 = static_cast<int>(std::min<int64_t>({p.dims[2], 256, kTmaBoxBytes / box_row_bytes}));
  // logical outer dims: 0 = d2 (box b2), 1 = d1, 2 = d0 (box 1)
  const int64_t ext[3] = {p.dims[2], p.dims[1], p.dims[0]};
  const cuuint32_t bx[3] = {cuuint32_t(b2), 1, 1};
  auto encode = [&](CUtensorMap* m, const void* ptr, const int64_t* stride, unsigned char* perm) {
    int64_t st[3] = {stride[2] * row, stride[1] * row, stride[0] * row};
    int64_t big = row * p.dims[3];
    for (int k = 0; k < 3; ++k)
      if (ext[k] > 1) big = std::max(big, st[k]);
    for (int k = 0; k < 3; ++k)
      if (ext[k] == 1) st[k] = big;  // any stride; keep the order monotonic
    int ord[3] = {0, 1, 2};
    std::stable_sort(ord, ord + 3, [&](int a, int b) { return st[a] < st[b]; });
    const cuuint64_t dims[5] = {cuuint64_t(p.hs_src), cuuint64_t(p.dims[3]), cuuint64_t(ext[ord[0]]),
                                cuuint64_t(ext[ord[1]]), cuuint64_t(ext[ord[2]])};
    const cuuint64_t str[4] = {cuuint64_t(row), cuuint64_t(st[ord[0]]), cuuint64_t(st[ord[1]]),
                               cuuint64_t(st[ord[2]])};
    for (int k = 0; k < 4; ++k)
      if (str[k] % 16 || str[k] >= (cuuint64_t(1) << 40) || str[k] == 0) return false;
    const cuuint32_t box[5] = {cuuint32_t(p.hs_src), cuuint32_t(b3), bx[ord[0]], bx[ord[1]], bx[ord[2]]};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    for (int k = 0; k < 3; ++k) perm[k] = static_cast<unsigned char>(ord[k]);
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(ptr), dims, str, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (!encode(&j.src, p.src, p.src_stride, j.ps) || !encode(&j.dst, p.dst, p.dst_stride, j.pd)) return false;
  j.b3 = b3;
  j.b2 = b2;
  j.n3 = static_cast<int>((p.dims[3] + b3 - 1) / b3);
  j.n2 = static_cast<int>((p.dims[2] + b2 - 1) / b2);
  j.n1 = static_cast<int>(p.dims[1]);
  j.bytes = static_cast<int>(box_row_bytes * b2);
  const int64_t boxes = int64_t(j.n3) * j.n2 * j.n1 * p.dims[0];
  if (boxes >= (int64_t(1) << 30)) return false;
  j.first = static_cast<int>(boxes);  // temporarily: this job's box count
  return true;
}

cudaError_t launch_tma(TmaParams& tp, int n, int num_sms, cudaStream_t stream) {
  int total = 0;
  for (int k = 0; k < n; ++k) {
    const int boxes = tp.job[k].first;
    tp.job[k].first = total;
    total += boxes;
  }
  tp.njobs = n;
  tp.total = total;
  if (!total) return cudaSuccess;
  constexpr int smem = kTmaSlots * kTmaBoxBytes + 1024;
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!(attr_done.load() & (uint64_t(1) << (dev & 63)))) {
    e = cudaFuncSetAttribute(reshard_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_done.fetch_or(uint64_t(1) << (dev & 63));
  }
  const int grid = std::max(1, std::min(num_sms, (total + 3) / 4));
  reshard_tma_kernel<<<grid, 32, smem, stream>>>(tp);
  return cudaGetLastError();
}
}  // namespace

// Several permutations in one launch: the TMA kernel when every one fits it
// (contiguous innermost dim, native head size), else one launch each.
cudaError_t launch_row_permute_multi(const RowPermute* ps, int n, int num_sms, cudaStream_t stream,
                                     int* launches) {
  static TmaParams tp;  // host staging (large); launches are issued from one thread per engine
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    bool tma = n <= kMaxTmaJobs && !dev_env("USPB_NO_TMA_RESHARD");
    for (int k = 0; tma && k < n; ++k) tma = to_tma_job(ps[k], tp.job[k]);
    if (tma) {
      if (launches) *launches = 1;
      return launch_tma(tp, n, num_sms, stream);
    }
  }
  for (int k = 0; k < n; ++k) {
    const cudaError_t e = launch_row_permute(ps[k], num_sms, stream);
    if (e != cudaSuccess) return e;
  }
  if (launches) *launches = n;
  return cudaSuccess;
}

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
