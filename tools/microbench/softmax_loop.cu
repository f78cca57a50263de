// Per-SMSP cost of the softmax exp loop (128 elements/row, 1 row/thread) for
// loop variants; W warps per SMSP. S values come from shared memory each
// iteration and P goes back to shared memory so nothing is hoisted.
#include <cstdio>
#include <cstdint>
#include "../../paper_2405_07719_b200/csrc/ptx_sm100.cuh"
using namespace uspb200::ptx;

template <int VAR>
__global__ void __launch_bounds__(512, 1) k(uint32_t* out, int iters) {
  __shared__ uint32_t sm[512 * 4];
  uint32_t s[128];
  for (int i = threadIdx.x; i < 512 * 4; i += blockDim.x) sm[i] = __float_as_uint(-0.01f * (i % 97));
  __syncthreads();
  float tot = 0.f;
  const float sl2 = 0.127f;
  long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 1) t0 = clock64();
#pragma unroll
    for (int i = 0; i < 128; ++i) s[i] = sm[(threadIdx.x + i * 13 + it) & 2047];
    const float neg = -1.f;
    const float2 sc2 = make_float2(sl2, sl2), nb2 = make_float2(neg, neg);
    float2 acc2 = make_float2(0.f, 0.f);
    float mxa = -INFINITY, mxb = -INFINITY;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const float a = __uint_as_float(s[2 * i]), c = __uint_as_float(s[2 * i + 1]);
      if (VAR & 1) { mxa = fmaxf(mxa, a); mxb = fmaxf(mxb, c); }
      const float2 x = ffma2(make_float2(a, c), sc2, nb2);
      float2 e;
      if ((VAR & 2) && (i & 7) >= 6) e = exp2_poly2(x);
      else { e.x = ex2(x.x); e.y = ex2(x.y); }
      acc2 = fadd2(acc2, e);
      s[i] = (VAR & 4) ? pack_bf16x2(e.x, e.y) : pack_bf16x2_pos(e.x, e.y);
    }
#pragma unroll
    for (int i = 0; i < 64; i += 16) sm[(threadIdx.x * 7 + i) & 2047] = s[i] ^ s[i + 5] ^ s[i + 11];
    tot += acc2.x + acc2.y + mxa + mxb;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(tot);
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (uint32_t)((t1 - t0) / (iters - 1));
}
template <int VAR> void run(int warps_per_smsp) {
  uint32_t* d; cudaMalloc(&d, (1 << 22) + 256);
  const int threads = 128 * warps_per_smsp;
  k<VAR><<<148, threads>>>(d, 4); cudaDeviceSynchronize();
  k<VAR><<<148, threads>>>(d, 64);
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t cyc; cudaMemcpy(&cyc, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
  printf("var=%d (max=%d poly=%d f2fp=%d) warps/SMSP=%d: %u cycles/iter -> %.0f cycles per 32-row x 128 tile per SMSP  %s\n",
         VAR, VAR & 1, (VAR >> 1) & 1, (VAR >> 2) & 1, warps_per_smsp, cyc, double(cyc) / warps_per_smsp, cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  for (int w : {1, 2, 4}) { run<0>(w); run<1>(w); run<2>(w); run<3>(w); run<4>(w); }
}
