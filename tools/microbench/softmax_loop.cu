// Cycles per 128-element softmax row-tile (exp + sum + pack) per SMSP, for
// variants of the inner loop of fa_fwd_sm100 (1 or 2 warps per SMSP).
#include <cstdio>
#include <cstdint>
#include "../../paper_2405_07719_b200/csrc/ptx_sm100.cuh"
using namespace uspb200::ptx;

template <int POLY, int PACK>  // PACK 0 = F2FP, 1 = PRMT
__global__ void k(uint32_t* out, int iters, float neg) {
  uint32_t s[128];
  for (int i = 0; i < 128; ++i) s[i] = __float_as_uint(-0.01f * (threadIdx.x % 7 + i));
  uint32_t acc = 0;
  const float sl2 = 0.127f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 128; ++i) asm volatile("" : "+r"(s[i]));
    const float2 sc2 = make_float2(sl2, sl2), nb2 = make_float2(neg, neg);
    float2 acc2 = make_float2(0.f, 0.f);
    uint32_t pk[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, nb2);
      float2 e;
      if ((i & 7) >= 8 - POLY) e = exp2_poly2(x);
      else { e.x = ex2(x.x); e.y = ex2(x.y); }
      acc2 = fadd2(acc2, e);
      pk[i] = PACK ? pack_bf16x2_pos(e.x, e.y) : pack_bf16x2(e.x, e.y);
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) { asm volatile("" : "+r"(pk[i])); acc ^= pk[i]; }
    acc += __float_as_uint(acc2.x + acc2.y);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (uint32_t)((t1 - t0) / iters);
}
template <int POLY, int PACK> void run(int warps) {
  uint32_t* d; cudaMalloc(&d, (1 << 22));
  k<POLY, PACK><<<148, 32 * warps>>>(d, 8, -1.f); cudaDeviceSynchronize();
  k<POLY, PACK><<<148, 32 * warps>>>(d, 256, -1.f); cudaDeviceSynchronize();
  uint32_t cyc; cudaMemcpy(&cyc, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
  // each warp does 32 rows x 128 elements per iteration; warps/4 warps share an SMSP
  printf("POLY=%d PACK=%s warps/SMSP=%d: %u cycles per iteration per warp -> %.0f cycles per 4096-elem SMSP tile\n",
         POLY, PACK ? "prmt" : "f2fp", warps / 4, cyc, double(cyc) / (warps / 4));
  cudaFree(d);
}
int main() {
  for (int w : {4, 8}) {
    run<0, 0>(w); run<0, 1>(w); run<2, 1>(w); run<3, 1>(w); run<4, 1>(w); run<2, 0>(w);
  }
}
