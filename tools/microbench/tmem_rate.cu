// TMEM load/store throughput on one SM (one CTA per SM, all SMs busy), alone
// and next to back-to-back tcgen05.mma (SS or TS, M = N = 128, bf16 -> fp32):
// does the compute warps' tcgen05.ld traffic (S / dP read-back) compete with
// the tensor pipe for TMEM bandwidth?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tmem_rate.cu -o tmem_rate
#include <cstdio>
#include <cstdint>
#include "../../paper_2405_07719_b200/csrc/ptx_sm100.cuh"
using namespace uspb200::ptx;

// LDW warps (multiple of 4) loop tcgen05.ld 32x32b.x32 (+ wait) over columns
// [0, 256) of their lane quarter; ST: tcgen05.st instead. MMA: 0 none, 1 SS,
// 2 TS — warp LDW issues 64 back-to-back MMAs (accumulator cols 256..383, TS A
// from cols 384..447) per commit while the loads run.
template <int LDW, bool ST, int MMA>
__global__ void __launch_bounds__(32 * (LDW + 1), 1) k(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ unsigned long long t_ld, t_mma;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 512);
  __syncthreads();
  fence_proxy_async_smem();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp < LDW) {
    const uint32_t lb = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    uint32_t acc = 0, r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = lane + i;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
      const uint32_t col = ((it * (LDW / 4) + warp / 4) & 7) * 32;
      if (ST) {
        tmem_st32(lb + col, r);
        tmem_st_wait();
      } else {
        tmem_ld32(lb + col, r);
        tmem_ld_wait(r);
        acc ^= r[0] ^ r[17] ^ r[31];
      }
    }
    const unsigned long long t1 = clock64();
    if (acc == 0x12345678u) out[1] = acc;
    if (threadIdx.x == 0) t_ld = t1 - t0;
  } else if (MMA != 0) {
    const uint32_t sa = smem_u32(base);
    const uint64_t ad = smem_desc_sw128(sa, 16, 1024);
    const uint64_t bd = smem_desc_sw128(sa + 32768, 16, 1024);
    const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
    const int batches = reps / 16 > 1 ? reps / 16 : 1;
    const unsigned long long t0 = clock64();
    for (int b = 0; b < batches; ++b) {
      if (elect_one()) {
        for (int i = 0; i < 64; ++i) {
          if (MMA == 2)
            mma_ts(tmem + 256, tmem + 384, bd, idesc, 1u);
          else
            mma_ss(tmem + 256, ad, bd, idesc, 1u);
        }
        mma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, b & 1);
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) t_mma = (t1 - t0) / (64ull * batches);
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = t_ld;
    out[2] = MMA ? t_mma : 0;
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int LDW, bool ST, int MMA>
void run(int reps) {
  unsigned long long* d;
  cudaMalloc(&d, 4 * 8);
  cudaMemset(d, 0, 32);
  auto kern = k<LDW, ST, MMA>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  kern<<<148, 32 * (LDW + 1), 80 * 1024>>>(d, 64);
  cudaDeviceSynchronize();
  kern<<<148, 32 * (LDW + 1), 80 * 1024>>>(d, reps);
  const cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double bytes = double(LDW) * reps * 32 * 32 * 4;
  printf("%s warps=%d mma=%s: %.1f B/clk/SM (%llu clk for %d x 4 KB per warp)  mma %llu clk/instr (alone 64)  %s\n",
         ST ? "STTM" : "LDTM", LDW, MMA == 0 ? "none" : (MMA == 1 ? "SS" : "TS"), bytes / double(h[0]), h[0], reps,
         h[2], cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  const int reps = 4096;
  run<4, false, 0>(reps);
  run<8, false, 0>(reps);
  run<16, false, 0>(reps);
  run<4, true, 0>(reps);
  run<8, true, 0>(reps);
  run<8, false, 1>(reps);
  run<8, false, 2>(reps);
  run<8, true, 1>(reps);
  run<8, true, 2>(reps);
  run<4, false, 1>(reps);
  run<4, false, 2>(reps);
  return 0;
}
