// reshard.cu — the Ulysses pack/unpack transposes (and head-size padding).
//
// Restates the data movement of scatter_heads_gather_seq /
// scatter_seq_gather_heads (reference src/usp/all_to_all_4d.cpp:27-39,
// 42-57, 75-87, 90-105) as one HBM-bound row-permutation kernel: every
// destination row (one head_size vector) is fetched from an affine source
// row index over four loop dimensions.
//
// Bulk path (every permutation the engine issues at a native head size: the
// innermost dimension is contiguous in source and destination, so a copy is
// a list of contiguous runs — (t, head range) blocks of heads/U * hs * 2
// bytes): the TMA bulk-copy engine moves the runs, global -> shared ->
// global (cp.async.bulk with mbarrier completion, then cp.async.bulk stores
// in bulk groups), from one issuing lane per warp with a ring of shared
// memory slots — no per-element instructions, and ONE launch for several
// tensors (Q, K and V packed together; every peer part of the direct
// exchange). Vector path (fallback): 32-bit index arithmetic, 16-byte
// loads with kUnroll in flight per thread. Head sizes that are not a
// multiple of 8 (or padding to a larger destination row) take the scalar
// path (small test shapes only).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "ptx_sm100.cuh"
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

// ----------------------------------------------------------------- bulk path
constexpr int kBulkWarps = 2;         // independent issuing lanes per CTA
constexpr int kBulkSlots = 16;        // shared-memory slots per warp
constexpr int kBulkSlot = 4096;       // bytes per slot
constexpr int kBulkAhead = 8;         // loads in flight ahead of the stores
constexpr int kMaxBulkJobs = 48;

struct BulkJob {
  const uint8_t* src;
  uint8_t* dst;
  uint64_t s0, s1, s2, t0, t1, t2;  // byte strides of the three outer dims
  uint32_t d1, d2;                  // run r = (i0 * d1 + i1) * d2 + i2
  uint32_t run_bytes;               // contiguous bytes per run (16-byte multiple)
  uint32_t group;                   // runs per item (run_bytes <= slot) ...
  uint32_t pieces;                  // ... or slot-sized pieces per run (run_bytes > slot)
  uint64_t runs;
  uint64_t first_item;              // prefix of items over the jobs
};
struct BulkParams {
  BulkJob job[kMaxBulkJobs];
  int njobs;
  uint64_t total_items;
};

__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(dst)),
               "r"(src_smem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_u32(uint32_t dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_smem),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Item i of the flattened job list -> (job, run range or piece).
struct Item {
  const BulkJob* j;
  uint64_t run;      // first run
  uint32_t nruns;    // runs in the item (group mode)
  uint32_t off, bytes;  // piece mode: byte offset inside the run, piece size
};
__device__ __forceinline__ Item locate_item(const BulkParams& p, uint64_t i) {
  int k = 0;
  while (k + 1 < p.njobs && p.job[k + 1].first_item <= i) ++k;
  const BulkJob& j = p.job[k];
  const uint64_t li = i - j.first_item;
  Item it;
  it.j = &j;
  if (j.pieces > 1) {
    it.run = li / j.pieces;
    const uint32_t pc = static_cast<uint32_t>(li % j.pieces);
    it.nruns = 1;
    it.off = pc * kBulkSlot;
    it.bytes = min(static_cast<uint32_t>(kBulkSlot), j.run_bytes - it.off);
  } else {
    it.run = li * j.group;
    const uint64_t left = j.runs - it.run;
    it.nruns = static_cast<uint32_t>(left < j.group ? left : j.group);
    it.off = 0;
    it.bytes = it.nruns * j.run_bytes;
  }
  return it;
}
__device__ __forceinline__ void run_addr(const BulkJob& j, uint64_t r, const uint8_t*& s, uint8_t*& d) {
  const uint64_t i2 = r % j.d2;
  const uint64_t q = r / j.d2;
  const uint64_t i1 = q % j.d1;
  const uint64_t i0 = q / j.d1;
  s = j.src + i0 * j.s0 + i1 * j.s1 + i2 * j.s2;
  d = j.dst + i0 * j.t0 + i1 * j.t1 + i2 * j.t2;
}

__global__ void __launch_bounds__(32 * kBulkWarps, 1) row_permute_bulk(const __grid_constant__ BulkParams p) {
  extern __shared__ __align__(128) uint8_t bulk_smem[];
  __shared__ __align__(8) uint64_t bars[kBulkWarps][kBulkSlots];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0) return;  // one issuing lane per warp
  uint64_t* bar = bars[warp];
  for (int s = 0; s < kBulkSlots; ++s) ptx::mbar_init(&bar[s], 1);
  ptx::fence_barrier_init();
  const uint32_t base = ptx::smem_u32(bulk_smem) + warp * kBulkSlots * kBulkSlot;
  const uint64_t lane_id = uint64_t(blockIdx.x) * kBulkWarps + warp;
  const uint64_t lanes = uint64_t(gridDim.x) * kBulkWarps;
  const uint64_t cnt = p.total_items > lane_id ? (p.total_items - lane_id + lanes - 1) / lanes : 0;
  for (uint64_t k = 0; k < cnt + kBulkAhead; ++k) {
    if (k < cnt) {  // load item k into slot k % S
      const uint32_t slot = static_cast<uint32_t>(k % kBulkSlots);
      // the slot's previous item (k - S) must have been read by its store;
      // stores issued so far: items < k - A, so at most S - A - 1 newer ones
      if (k >= kBulkSlots) bulk_wait_read<kBulkSlots - kBulkAhead - 1>();
      const Item it = locate_item(p, lane_id + k * lanes);
      ptx::mbar_arrive_expect_tx(&bar[slot], it.bytes);
      uint32_t dst = base + slot * kBulkSlot;
      for (uint32_t r = 0; r < it.nruns; ++r) {
        const uint8_t* s;
        uint8_t* d;
        run_addr(*it.j, it.run + r, s, d);
        const uint32_t b = it.j->pieces > 1 ? it.bytes : it.j->run_bytes;
        bulk_g2s_u32(dst, s + it.off, b, &bar[slot]);
        dst += b;
      }
    }
    if (k >= kBulkAhead && k - kBulkAhead < cnt) {  // store item k - A
      const uint64_t m = k - kBulkAhead;
      const uint32_t slot = static_cast<uint32_t>(m % kBulkSlots);
      ptx::mbar_wait(&bar[slot], static_cast<uint32_t>((m / kBulkSlots) & 1));
      const Item it = locate_item(p, lane_id + m * lanes);
      uint32_t src = base + slot * kBulkSlot;
      for (uint32_t r = 0; r < it.nruns; ++r) {
        const uint8_t* s;
        uint8_t* d;
        run_addr(*it.j, it.run + r, s, d);
        const uint32_t b = it.j->pieces > 1 ? it.bytes : it.j->run_bytes;
        bulk_s2g(d + it.off, src, b);
        src += b;
      }
      bulk_commit();
    }
  }
  bulk_wait_all();
}

int64_t max_row(const RowPermute& p, const int64_t* stride) {
  int64_t m = 0;
  for (int i = 0; i < 4; ++i) m += (p.dims[i] - 1) * stride[i];
  return m;
}


// RowPermute -> bulk job: the innermost dim must be contiguous in both
// tensors (then it and any further contiguous dims form one run).
bool to_bulk_job(const RowPermute& p, BulkJob& j) {
  if (p.hs_src != p.hs_dst || (p.hs_src * 2) % 16 != 0) return false;
  if (p.src_stride[3] != 1 || p.dst_stride[3] != 1) return false;
  const int64_t row = p.hs_src * 2;
  int64_t run_rows = p.dims[3];
  int outer = 2;  // dims[0..outer] are loops
  while (outer >= 0 && p.src_stride[outer] == run_rows && p.dst_stride[outer] == run_rows) {
    run_rows *= p.dims[outer];
    --outer;
  }
  int64_t d[3] = {1, 1, 1}, ss[3] = {0, 0, 0}, ts[3] = {0, 0, 0};
  for (int k = 0; k <= outer; ++k) {  // right-align the remaining loop dims into d[0..2]
    const int slot = 2 - (outer - k);
    d[slot] = p.dims[k];
    ss[slot] = p.src_stride[k] * row;
    ts[slot] = p.dst_stride[k] * row;
  }
  const int64_t run_bytes = run_rows * row;
  if (run_bytes <= 0 || run_bytes > (int64_t(1) << 30)) return false;
  for (int k = 0; k < 3; ++k)
    if (ss[k] % 16 || ts[k] % 16) return false;
  if (reinterpret_cast<uintptr_t>(p.src) % 16 || reinterpret_cast<uintptr_t>(p.dst) % 16) return false;
  j.src = static_cast<const uint8_t*>(p.src);
  j.dst = static_cast<uint8_t*>(p.dst);
  j.s0 = ss[0], j.s1 = ss[1], j.s2 = ss[2];
  j.t0 = ts[0], j.t1 = ts[1], j.t2 = ts[2];
  j.d1 = static_cast<uint32_t>(d[1]);
  j.d2 = static_cast<uint32_t>(d[2]);
  j.run_bytes = static_cast<uint32_t>(run_bytes);
  j.runs = static_cast<uint64_t>(d[0] * d[1] * d[2]);
  if (run_bytes <= kBulkSlot) {
    j.group = static_cast<uint32_t>(kBulkSlot / run_bytes);
    j.pieces = 1;
  } else {
    j.group = 1;
    j.pieces = static_cast<uint32_t>((run_bytes + kBulkSlot - 1) / kBulkSlot);
  }
  return true;
}

cudaError_t launch_bulk(const BulkJob* jobs, int n, int num_sms, cudaStream_t stream) {
  BulkParams bp{};
  uint64_t items = 0;
  for (int k = 0; k < n; ++k) {
    bp.job[k] = jobs[k];
    bp.job[k].first_item = items;
    items += jobs[k].pieces > 1 ? jobs[k].runs * jobs[k].pieces : (jobs[k].runs + jobs[k].group - 1) / jobs[k].group;
  }
  bp.njobs = n;
  bp.total_items = items;
  if (!items) return cudaSuccess;
  constexpr int smem = kBulkWarps * kBulkSlots * kBulkSlot;
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!(attr_done.load() & (uint64_t(1) << (dev & 63)))) {
    e = cudaFuncSetAttribute(row_permute_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_done.fetch_or(uint64_t(1) << (dev & 63));
  }
  const uint64_t lanes_needed = (items + 3) / 4;  // >= 4 items per issuing lane
  const int grid = static_cast<int>(std::min<uint64_t>(num_sms, (lanes_needed + kBulkWarps - 1) / kBulkWarps));
  row_permute_bulk<<<grid > 0 ? grid : 1, 32 * kBulkWarps, smem, stream>>>(bp);
  return cudaGetLastError();
}

}  // namespace

// Several permutations in one launch: the bulk kernel when every one
// qualifies (contiguous innermost dim, 16-byte runs, native head size),
// else one launch each.
cudaError_t launch_row_permute_multi(const RowPermute* ps, int n, int num_sms, cudaStream_t stream,
                                     int* launches) {
  BulkJob jobs[kMaxBulkJobs];
  bool bulk = n <= kMaxBulkJobs && !std::getenv("USPB_NO_BULK");
  for (int k = 0; bulk && k < n; ++k) bulk = to_bulk_job(ps[k], jobs[k]);
  if (bulk) {
    if (launches) *launches = 1;
    return launch_bulk(jobs, n, num_sms, stream);
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
