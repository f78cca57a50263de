// Throughput of the softmax building blocks on one SM (1..4 warps per SMSP).
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#define N 4096
__global__ void k_ex2_f32(float* out, int iters) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i]; out[threadIdx.x] = s;
}
__global__ void k_ex2_f16x2(float* out, int iters) {
  unsigned a[8]; for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(-0.001f*threadIdx.x, -0.002f*i); a[i] = *(unsigned*)&h; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += __half2float(*(__half*)&a[i]); out[threadIdx.x] = s;
}
__global__ void k_ex2_bf16x2(float* out, int iters) {
  unsigned a[8]; for (int i = 0; i < 8; ++i) { __nv_bfloat162 h = __floats2bfloat162_rn(-0.001f*threadIdx.x, -0.002f*i); a[i] = *(unsigned*)&h; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += (float)(*(__nv_bfloat16*)&a[i]); out[threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, int iters) {
  float2 a[8]; for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x, i);
  const float2 b = make_float2(0.999f, 0.998f), c = make_float2(0.001f, 0.002f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("{.reg .b64 x,y,z; mov.b64 x,{%0,%1}; mov.b64 y,{%2,%3}; mov.b64 z,{%4,%5}; fma.rn.f32x2 x,x,y,z; mov.b64 {%0,%1},x;}" : "+f"(a[i].x), "+f"(a[i].y) : "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y; out[threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  float b = out[1000], c = out[1001];
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i]; out[threadIdx.x] = s;
}
__global__ void k_f2fp(float* out, int iters) {
  float a[8]; unsigned r[8]; for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; r[i] = 0; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { unsigned t; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(t) : "f"(a[i]), "f"(a[(i+1)&7])); r[i] ^= t; a[i] = __uint_as_float(r[i] | 0x3f800000u); }
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += r[i]; out[threadIdx.x] = s;
}
template <class K> void run(const char* name, K kern, int warps) {
  float* d; cudaMalloc(&d, 1 << 16); cudaMemset(d, 0, 1 << 16);
  int iters = 4096;
  kern<<<148, 32 * warps>>>(d, 16); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); kern<<<148, 32 * warps>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double instr_per_sm = double(iters) * 8 * warps;  // warp-instructions per SM
  double cyc = ms * 1e-3 * clk * 1e3;  // at max clock (approx)
  printf("%-10s warps/SM=%2d  %.3f ms  ~%.2f cyc per warp-instr per SM (at %d MHz)  lanes/clk/SM=%.1f\n", name, warps, ms,
         cyc / instr_per_sm, clk / 1000, instr_per_sm * 32 / cyc);
  cudaFree(d);
}
int main() {
  for (int w : {4, 8, 16}) {
    run("ex2.f32", k_ex2_f32, w); run("ex2.f16x2", k_ex2_f16x2, w); run("ex2.bf16x2", k_ex2_bf16x2, w);
    run("ffma2", k_ffma2, w); run("ffma", k_ffma, w); run("f2fp", k_f2fp, w);
  }
}
