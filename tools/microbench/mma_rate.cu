// Back-to-back tcgen05.mma issue rate on one SM (one CTA per SM, all SMs busy):
// cycles per instruction for SS / TS, N in {64,128,256}, M = 128, bf16 -> fp32.
#include <cstdio>
#include <cstdint>
#include "../../paper_2405_07719_b200/csrc/ptx_sm100.cuh"
using namespace uspb200::ptx;

// MODE 0: 64 back-to-back MMAs per commit; MODE 1: batches of 8 MMAs each
// followed by commit + tcgen05.fence::after_thread_sync; MODE 2: batches of 8
// with commit + a wait on an already-complete mbarrier + fence.
template <int N, bool TS, int MODE = 0>
__global__ void __launch_bounds__(256, 1) k(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&tslot, 512);
  __syncthreads();
  fence_proxy_async_smem();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if ((MODE == 3 || MODE == 4) && warp >= 4) {
    // background shared-memory traffic: 4 warps of 16-byte stores / loads
    uint4* region = reinterpret_cast<uint4*>(base + 65536);
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    for (int i = 0; i < 20000; ++i) {
      const int idx = ((threadIdx.x - 128) + i * 128) & 1023;
      if (MODE == 3) region[idx] = v;
      else { v.x ^= region[idx].x; }
    }
    if (v.x == 12345) out[1] = v.y;
  }
  if (warp == 0) {
    const uint32_t sa = smem_u32(base);
    const uint64_t ad = smem_desc_sw128(sa, 16, 1024);
    const uint64_t bd = smem_desc_sw128(sa + 32768, 16, 1024);
    const uint32_t idesc = idesc_bf16_f32(128, N, 0, 0);
    unsigned long long t0 = 0, t1 = 0;
    for (int r = 0; r < reps; ++r) {
      if (r == 1) t0 = clock64();
      if (MODE == 0 || MODE >= 3) {
        if (elect_one()) {
          for (int i = 0; i < 64; ++i) {
            if (TS) mma_ts(tmem + 256, tmem + 0, bd, idesc, 1u);
            else mma_ss(tmem + 256, ad, bd, idesc, 1u);
          }
          mma_commit(&bar);
        }
        __syncwarp();
      } else {
        for (int b = 0; b < 8; ++b) {
          if (MODE == 2 && b > 0) mbar_wait(&bar2, 0);  // already complete after first arrive
          tc_fence_after();
          if (elect_one()) {
            for (int i = 0; i < 8; ++i) {
              if (TS) mma_ts(tmem + 256, tmem + 0, bd, idesc, 1u);
              else mma_ss(tmem + 256, ad, bd, idesc, 1u);
            }
            if (b == 7) mma_commit(&bar);
            else if (MODE == 2 && r == 0 && b == 0) mbar_arrive(&bar2);
            else mma_commit(&bar2 + 0 * b);
          }
          __syncwarp();
        }
      }
      mbar_wait(&bar, r & 1);
    }
    t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / (64ull * (reps - 1));
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}
template <int N, bool TS, int MODE = 0> void run() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  auto kern = k<N, TS, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kern<<<148, 256, 100 * 1024>>>(d, 4); cudaDeviceSynchronize();
  kern<<<148, 256, 100 * 1024>>>(d, 40);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double flop = 2.0 * 128 * N * 16;
  printf("mode %d %s N=%3d: %llu cycles per MMA (theory %d) -> %.0f FLOP/clk/SM (%s)\n", MODE, TS ? "TS" : "SS", N, h[0], 128 * N / 256,
         flop / h[0], cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  run<64, false>(); run<128, false>(); run<256, false>();
  run<64, true>(); run<128, true>(); run<256, true>();
  run<128, false, 1>(); run<128, true, 1>(); run<128, false, 2>(); run<128, true, 2>();
  run<128, false, 3>(); run<128, true, 3>(); run<128, false, 4>(); run<128, true, 4>();
}
