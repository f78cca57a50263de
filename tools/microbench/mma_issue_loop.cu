// The dQ kernel's MMA-warp issue pattern in isolation: per "tile"
//   wait A -> 8 SS MMAs -> commit s_full -> wait B -> 8 SS MMAs -> commit
//   dp_full, commit v_empty -> wait C -> 4 TS MMAs -> wait D -> 4 TS MMAs ->
//   commit k_empty
// with every wait on a phase that is already complete (the issuing thread
// arrives on it first), against 24 back-to-back MMAs. The difference is the
// issue-stream cost of the waits and commits alone (no producer/consumer).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_issue_loop.cu -o mma_issue_loop
#include <cstdio>
#include <cstdint>
#include "../../paper_2405_07719_b200/csrc/ptx_sm100.cuh"
using namespace uspb200::ptx;

// MODE 0: 24 MMAs back to back per tile; 1: the dQ pattern; 2: pattern
// without waits; 3-5: the dQ pattern while 8 "compute" warps loop on their
// own TMEM columns (3: tcgen05.ld/st only, 4: ld/st + ex2/FFMA2 on the
// values, 5: ex2/FFMA2 only) — what the real kernels run next to the MMAs.
template <int MODE>
__global__ void __launch_bounds__(288, 1) k(unsigned long long* out, int tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t tslot;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) stop = 0;
  if (warp == 0) tmem_alloc(&tslot, 512);
  __syncthreads();
  fence_proxy_async_smem();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp > 0) {  // background compute warps 1..8 on TMEM columns 0..127 of their lane quarter
    if (MODE >= 3) {
      const int q = (warp - 1) & 3, h = (warp - 1) >> 2;
      const uint32_t lb = tmem + (static_cast<uint32_t>(q * 32) << 16) + h * 64;
      uint32_t r[64];
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 64; ++i) r[i] = __float_as_uint(float(lane + i) * 1e-3f);
      while (!stop) {
        if (MODE != 5) {
          tmem_ld32(lb, r);
          tmem_ld32(lb + 32, r + 32);
          tmem_ld_wait(r);
          tmem_ld_wait(r + 32);
        }
        if (MODE != 3) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 x = ffma2(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])),
                                   make_float2(0.5f, 0.5f), make_float2(-1.f, -1.f));
            r[2 * i] = __float_as_uint(ex2(x.x));
            r[2 * i + 1] = __float_as_uint(ex2(x.y));
          }
        }
        if (MODE != 5) {
          tmem_st32(lb, r);
          tmem_st_wait();
        }
        acc += __uint_as_float(r[0]) + __uint_as_float(r[63]);
      }
      if (acc == 1234.5f) out[1] = 1;
    }
    __syncthreads();
    return;
  }
  const uint32_t sa = smem_u32(base);
  const uint64_t ad = smem_desc_sw128(sa, 16, 1024);
  const uint64_t bd = smem_desc_sw128(sa + 32768, 16, 1024);
  const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
  auto ss8 = [&](uint32_t d) {
    if (elect_one())
      for (int i = 0; i < 8; ++i) mma_ss(tmem + d, ad, bd, idesc, i > 0 ? 1u : 0u);
    __syncwarp();
  };
  auto ts4 = [&]() {
    if (elect_one())
      for (int i = 0; i < 4; ++i) mma_ts(tmem + 384, tmem + 0, bd, idesc, 1u);
    __syncwarp();
  };
  auto wait_done = [&](int b, int t) {  // a phase completed by this thread's own arrive
    if (MODE == 1 || MODE >= 3) {
      if (threadIdx.x == 0) mbar_arrive(&bars[b]);
      mbar_wait(&bars[b], t & 1);
      tc_fence_after();
    }
  };
  auto commit = [&](int b) {
    if (MODE != 0) {
      if (elect_one()) mma_commit(&bars[4 + b]);
      __syncwarp();
    }
  };
  unsigned long long t0 = 0;
  for (int t = 0; t < tiles; ++t) {
    if (t == 2) t0 = clock64();
    wait_done(0, t);
    ss8(128);
    commit(0);
    wait_done(1, t);
    ss8(256);
    commit(1);
    commit(2);
    wait_done(2, t);
    ts4();
    wait_done(3, t);
    ts4();
    commit(3);
  }
  // drain: wait for the last commit of barrier 7 (or a fresh one in mode 0)
  if (elect_one()) mma_commit(&bars[7]);
  __syncwarp();
  mbar_wait(&bars[7], MODE == 0 ? 0 : (tiles & 1));
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / (tiles - 2);
  if (threadIdx.x == 0) stop = 1;
  __syncthreads();
  tmem_dealloc(tmem, 512);
}

template <int MODE>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  auto kern = k<MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kern<<<148, 288, 100 * 1024>>>(d, 8);
  cudaDeviceSynchronize();
  kern<<<148, 288, 100 * 1024>>>(d, 202);
  const cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const char* name[] = {"24 MMAs back to back", "dQ pattern (4 completed waits, 5 commits)", "dQ pattern, commits only",
                        "dQ pattern + 8 warps TMEM ld/st", "dQ pattern + 8 warps TMEM ld/st + ex2/FFMA2",
                        "dQ pattern + 8 warps ex2/FFMA2"};
  printf("%-44s: %llu clk per tile (24 x 66 = 1584)  %s\n", name[MODE], h, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>();
  run<2>();
  run<1>();
  run<3>();
  run<4>();
  run<5>();
  return 0;
}
