// Global fp32 reduction throughput per SM for the fused backward's dQ drain
// (development aid): one CTA per SM, W warps, each "tile" reduces 64 KB
// (128 rows x 128 fp32, rows 16 KB apart as dQ rows of 32 heads x 128).
//   mode 0: red.add.f32, lane = column (32 consecutive floats = one 128 B
//           line per instruction), 128 rows per warp-quarter  [the kernel's drain]
//   mode 1: red.add.v4.f32, lane = row (16 B per lane, 32 rows per instruction)
//   mode 2: red.add.v4.f32, lanes cover one row's 512 B (4 lines per instruction)
//   mode 3: cp.reduce.async.bulk.add.f32 from shared memory, 512 B per row
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/red_rate red_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void red1(float* a, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void red4(float* a, float v) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %1, %1, %1};" ::"l"(a), "f"(v) : "memory");
}

template <int MODE>
__global__ void k(float* buf, int iters, int nqt, int warps_per_tile, unsigned long long* cyc) {
  extern __shared__ __align__(128) float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const size_t row_stride = 32 * 128;  // floats
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) sm[i] = 1.f;
  __syncthreads();
  unsigned long long t0 = clock64();
  const float v = 1.0f;
  for (int it = 0; it < iters; ++it) {
    // tile (head, q tile) of this iteration
    const int h = blockIdx.x % 32, qt = (blockIdx.x / 32 + it) % nqt;
    float* tile = buf + (static_cast<size_t>(qt) * 128 * 32 + h) * 128;
    // each warp takes 1/nw of the tile's work
    if (MODE == 0) {
      // 4 column groups x 128 rows; warp w: column group w % 4, rows split over nw/4 warps
      const int cg = warp & 3, part = warp >> 2, parts = nw / 4;
      for (int j = part; j < 128; j += parts) red1(tile + j * row_stride + cg * 32 + lane, v);
    } else if (MODE == 1) {
      const int rows_per = 128 / nw;
      for (int k4 = 0; k4 < 32; ++k4)
        for (int rr = 0; rr < rows_per; rr += 32)
          red4(tile + (warp * rows_per + rr + lane) * row_stride + k4 * 4, v);
    } else if (MODE == 2) {
      const int rows_per = 128 / nw;
      for (int j = 0; j < rows_per; ++j) red4(tile + (warp * rows_per + j) * row_stride + lane * 4, v);
    } else {
      const int rows_per = 128 / nw;
      if (lane == 0) {
        for (int j = 0; j < rows_per; ++j) {
          const float* src = sm + (warp * rows_per + j) * 128;
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;" ::"l"(
                           tile + (warp * rows_per + j) * row_stride),
                       "r"(static_cast<uint32_t>(__cvta_generic_to_shared(src)))
                       : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      }
      __syncwarp();
    }
  }
  if (MODE == 3 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int nsm = 148;
  for (int big = 0; big < 2; ++big) {
    const int nqt = big ? 512 : 16;  // 16: 32 MB (L2-resident); 512: 1 GB
    const size_t n = static_cast<size_t>(nqt) * 128 * 32 * 128;
    float* buf;
    cudaMalloc(&buf, n * 4);
    cudaMemset(buf, 0, n * 4);
    unsigned long long* cyc;
    cudaMalloc(&cyc, nsm * 8);
    for (int mode = 0; mode < 4; ++mode)
      for (int nw : {4, 8}) {
        const int iters = 200;
        auto launch = [&]() {
          const int smem = 128 * 128 * 4;
          if (mode == 0) { cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<0><<<nsm, nw * 32, smem>>>(buf, iters, nqt, 0, cyc); }
          if (mode == 1) { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<1><<<nsm, nw * 32, smem>>>(buf, iters, nqt, 0, cyc); }
          if (mode == 2) { cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<2><<<nsm, nw * 32, smem>>>(buf, iters, nqt, 0, cyc); }
          if (mode == 3) { cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<3><<<nsm, nw * 32, smem>>>(buf, iters, nqt, 0, cyc); }
        };
        launch();
        cudaDeviceSynchronize();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long h[148];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < nsm; ++i) avg += h[i];
        avg /= nsm;
        const double bytes = double(nsm) * iters * 65536.0;
        printf("%s mode %d warps %d: %.3f ms, %.2f TB/s, %.0f clk per 64 KB tile per SM (%.1f B/clk/SM) err=%s\n",
               big ? "1GB " : "32MB", mode, nw, ms, bytes / ms / 1e9, avg / iters, 65536.0 * iters / avg,
               cudaGetErrorString(cudaGetLastError()));
      }
    cudaFree(buf);
    cudaFree(cyc);
  }
  return 0;
}
