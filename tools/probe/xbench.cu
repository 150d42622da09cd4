// Exchange-layout microbenchmark for the 32x32 warp transpose of 16-B elements.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__device__ __forceinline__ int wr_idx(int k, int lane) {   // writer: lane holds row element k
  if (MODE == 0) return k * 33 + lane;                // stride-33 padding
  if (MODE == 1) return k * 32 + (lane ^ k);          // XOR swizzle
  if (MODE == 2) return k * 32 + ((lane + k) & 31);   // rotation
  return k * 34 + lane;                               // stride 34
}
template <int MODE>
__device__ __forceinline__ int rd_idx(int lane, int l) {   // reader: lane = k, reads element l
  if (MODE == 0) return lane * 33 + l;
  if (MODE == 1) return lane * 32 + (l ^ lane);
  if (MODE == 2) return lane * 32 + ((l + lane) & 31);
  return lane * 34 + l;
}
template <int MODE>
__global__ void kx(double2* out, int iters) {
  __shared__ double2 xs[2][32 * 34];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = make_double2(lane + r, r);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 32; ++k) xs[w][wr_idx<MODE>(k, lane)] = v[k];
    __syncwarp();
#pragma unroll
    for (int l = 0; l < 32; ++l) v[l] = xs[w][rd_idx<MODE>(lane, l)];
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r].x += 1.0;
  }
  double2 s = make_double2(0, 0);
#pragma unroll
  for (int r = 0; r < 32; ++r) { s.x += v[r].x; s.y += v[r].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE> void run(double2* out) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  kx<MODE><<<148 * 4, 64>>>(out, 10);
  cudaEventRecord(a); kx<MODE><<<148 * 4, 64>>>(out, 1000); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double bytes = 148.0 * 4 * 64 * 1000 * 32 * 16 * 2;
  printf("mode %d: %.3f ms, smem %.1f TB/s (%.0f B/clk/SM at 1.965 GHz)\n", MODE, ms, bytes / ms / 1e9, bytes / (ms * 1e-3) / 148 / 1.965e9);
}
int main() { double2* out; cudaMalloc(&out, 1 << 24); run<0>(out); run<1>(out); run<2>(out); run<3>(out); return 0; }
