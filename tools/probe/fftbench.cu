// Microbenchmark: warp_fft1024 throughput in isolation (data in registers + warp smem region).
#include <cstdio>
#include "../../paper_2407_16559_b200/csrc/fft.cuh"
using namespace agk;
template <int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) kbench(double2* out, const double2* gtw, int iters) {
  extern __shared__ double2 sm[];
  double2* tw = sm + WARPS * (kXS + 1);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tw[i] = gtw[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = make_double2(lane + r, r - lane);
  for (int it = 0; it < iters; ++it) {
    warp_fft1024<-1, false>(v, sm + w * (kXS + 1), tw, lane);
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = make_double2(v[r].x * 1e-3, v[r].y * 1e-3);
  }
  double2 s = czero();
#pragma unroll
  for (int r = 0; r < 32; ++r) s = cadd(s, v[r]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int WARPS, int MINB>
void run(double2* out, double2* tw, int blocks, size_t extra = 0) {
  size_t smem = (WARPS * (kXS + 1) + 1024) * sizeof(double2) + extra;
  cudaFuncSetAttribute(kbench<WARPS, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 200;
  kbench<WARPS, MINB><<<blocks, WARPS * 32, smem>>>(out, tw, 10);
  cudaEventRecord(a);
  kbench<WARPS, MINB><<<blocks, WARPS * 32, smem>>>(out, tw, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ffts = (double)blocks * WARPS * iters;
  double flops = ffts * 5.0 * 1024 * 10;
  printf("warps/blk %d minb %d blocks %d: %.3f ms, %.1f Mfft/s, %.2f TFLOP/s (5NlogN) err=%s\n", WARPS, MINB, blocks, ms,
         ffts / ms / 1e3, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double2 *out, *tw; cudaMalloc(&out, 1 << 26); cudaMalloc(&tw, 1024 * 16);
  double2 h[1024];
  for (int k = 0; k < 32; ++k) for (int l = 0; l < 32; ++l) { double a = -2 * 3.141592653589793 * l * k / 1024; h[k * 32 + l] = make_double2(cos(a), sin(a)); }
  cudaMemcpy(tw, h, sizeof(h), cudaMemcpyHostToDevice);
  run<8, 1>(out, tw, 148);
  run<4, 1>(out, tw, 148, 120000);   // 1 block of 4 warps per SM
  run<2, 1>(out, tw, 148, 160000);   // 2 warps per SM
  run<4, 2>(out, tw, 296);
  return 0;
}
