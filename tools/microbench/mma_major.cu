// tcgen05.mma rate by B-operand major-ness: TS and SS, M = N = 128,
// bf16 -> fp32, B K-major (S = Q K^T style) vs MN-major (dQ += dS K,
// dV += P^T dO, dK += dS^T Q in the backward kernels), back to back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_major.cu -o mma_major
#include <cstdio>
#include <cstdint>
#include "../../paper_2405_07719_b200/csrc/ptx_sm100.cuh"
using namespace uspb200::ptx;

template <bool TS, bool BMN>
__global__ void __launch_bounds__(32, 1) k(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tmem_alloc(&tslot, 512);
  __syncwarp();
  fence_proxy_async_smem();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t sa = smem_u32(base);
  const uint64_t ad = smem_desc_sw128(sa, 16, 1024);
  // B: K-major (LBO unused for SW128 K-major) or MN-major over two 64-column
  // sub-blocks of 16 KB (the kernels' layout: LBO = sub-block stride)
  const uint64_t bd = BMN ? smem_desc_sw128(sa + 32768, 128 * 128, 1024) : smem_desc_sw128(sa + 32768, 16, 1024);
  const uint32_t idesc = idesc_bf16_f32(128, 128, 0, BMN ? 1u : 0u);
  unsigned long long t0 = 0;
  for (int r = 0; r < reps; ++r) {
    if (r == 1) t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < 64; ++i) {
        if (TS)
          mma_ts(tmem + 256, tmem + 0, bd, idesc, 1u);
        else
          mma_ss(tmem + 256, ad, bd, idesc, 1u);
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, r & 1);
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / (64ull * (reps - 1));
  __syncwarp();
  tmem_dealloc(tmem, 512);
}

template <bool TS, bool BMN>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  auto kern = k<TS, BMN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kern<<<148, 32, 100 * 1024>>>(d, 4);
  cudaDeviceSynchronize();
  kern<<<148, 32, 100 * 1024>>>(d, 60);
  const cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%s B %s-major: %llu clk/MMA (floor 64)  %s\n", TS ? "TS" : "SS", BMN ? "MN" : "K ", h, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<false, false>();
  run<false, true>();
  run<true, false>();
  run<true, true>();
  return 0;
}
