// tcgen05.mma rate (M = N = 128, bf16 -> fp32, SS or TS) while another warp
// streams bulk copies (cp.async.bulk global -> shared, like the kernels' TMA
// tile loads) into a separate shared-memory region: do TMA writes compete
// with the MMA operand reads for shared-memory bandwidth?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_smem_contention.cu -o mma_smem_contention
#include <cstdio>
#include <cstdint>
#include "../../paper_2405_07719_b200/csrc/ptx_sm100.cuh"
using namespace uspb200::ptx;

// LOAD_KB: bytes per bulk copy (KB), 0 = no background copies; INFLIGHT copies
// kept in flight by the loader warp.
template <bool TS, int LOAD_KB, int INFLIGHT>
__global__ void __launch_bounds__(64, 1) k(unsigned long long* out, const uint8_t* src, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, lbar[4];
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&lbar[i], 1);
    fence_barrier_init();
    stop = 0;
  }
  if (warp == 0) tmem_alloc(&tslot, 512);
  __syncthreads();
  fence_proxy_async_smem();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1) {
    if (LOAD_KB > 0 && threadIdx.x == 32) {
      uint8_t* dst = base + 65536;  // 64 KB of operands below, copies above
      const uint32_t bytes = LOAD_KB * 1024;
      unsigned long long moved = 0;
      uint32_t ph[4] = {0, 0, 0, 0};
      for (int i = 0; i < INFLIGHT; ++i) {
        mbar_arrive_expect_tx(&lbar[i], bytes);
        bulk_g2s(dst + i * bytes, src + (size_t(blockIdx.x) * 8 + i) * bytes, bytes, &lbar[i]);
      }
      const unsigned long long t0 = clock64();
      for (int it = 0; !stop; ++it) {
        const int s = it % INFLIGHT;
        mbar_wait(&lbar[s], ph[s]);
        ph[s] ^= 1;
        moved += bytes;
        mbar_arrive_expect_tx(&lbar[s], bytes);
        bulk_g2s(dst + s * bytes, src + (size_t(blockIdx.x) * 8 + s) * bytes, bytes, &lbar[s]);
      }
      for (int s = 0; s < INFLIGHT; ++s) mbar_wait(&lbar[s], ph[s]);
      const unsigned long long t1 = clock64();
      if (blockIdx.x == 0) out[1] = static_cast<unsigned long long>(double(moved) / double(t1 - t0) * 100.0);
    }
  } else {
    const uint32_t sa = smem_u32(base);
    const uint64_t ad = smem_desc_sw128(sa, 16, 1024);
    const uint64_t bd = smem_desc_sw128(sa + 32768, 16, 1024);
    const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
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
    if (threadIdx.x == 0) {
      if (blockIdx.x == 0) out[0] = (t1 - t0) / (64ull * (reps - 1));
      stop = 1;
    }
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <bool TS, int LOAD_KB, int INFLIGHT>
void run(const uint8_t* src) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  auto kern = k<TS, LOAD_KB, INFLIGHT>;
  const int smem = 1024 + 65536 + 4 * 32 * 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<148, 64, smem>>>(d, src, 4);
  cudaDeviceSynchronize();
  kern<<<148, 64, smem>>>(d, src, 200);
  const cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s MMA with %2d KB x %d bulk copies in flight: %llu clk/MMA (alone 66-67); copies %.1f B/clk/SM  %s\n",
         TS ? "TS" : "SS", LOAD_KB, INFLIGHT, h[0], h[1] / 100.0, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, size_t(148) * 8 * 32 * 1024);
  cudaMemset(src, 1, size_t(148) * 8 * 32 * 1024);
  run<false, 0, 1>(src);
  run<false, 16, 2>(src);
  run<false, 32, 2>(src);
  run<false, 32, 4>(src);
  run<true, 0, 1>(src);
  run<true, 32, 2>(src);
  run<true, 32, 4>(src);
  return 0;
}
