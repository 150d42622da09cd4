// Microbenchmark: throughput of the warp-synchronous 1024-point fp64 transform (warp_fft1024,
// fft.cuh) and of its pieces, per SM, against the number of resident warps. Data stays in
// registers; every warp repeats the transform in place `iters` times. Prints cycles per transform
// per SM (the figure the column and row passes are built from: 221 transforms per SM per pass at
// config 4) and fp64 DADD latency/throughput for reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o wfft wfft.cu
#include <cmath>
#include <cstdio>
#include <vector>
#include "../../paper_2407_16559_b200/csrc/fft.cuh"
using namespace agk;

constexpr int kX = 33;  // exchange stride

template <int MODE>
__global__ void __launch_bounds__(256, 1) kfft(double2* out, const double2* tw_g, int iters, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* tw = sm;
  double2* xs = sm + 1024 + (threadIdx.x >> 5) * 32 * kX;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tw[i] = tw_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = make_double2(1e-3 * (lane + r), 1e-3 * (r - lane));
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      warp_fft1024<-1, false, true>(v, xs, tw, lane);  // full transform, recurrence twiddles
    } else if (MODE == 1) {
      warp_fft1024<-1, false, false>(v, xs, tw, lane);  // table twiddles
    } else if (MODE == 2) {
      Dft<32, -1>::run(v);  // one radix-32 register DFT
    } else if (MODE == 3) {
      Dft<32, -1>::run(v);
      Dft<32, -1>::run(v);  // both register DFTs, no twiddles, no exchange
    }
    // keep magnitudes bounded
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = make_double2(v[r].x * (1.0 / 1024), v[r].y * (1.0 / 1024));
  }
  const long long t1 = clock64();
  if (lane == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
  double2 s = make_double2(0, 0);
#pragma unroll
  for (int r = 0; r < 32; ++r) s = cadd(s, v[r]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void kdadd(double* out, int iters, int ilp, long long* cyc) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  const double b = 1e-9;
  const long long t0 = clock64();
  if (ilp == 1) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 16; ++u) a[0] = a[0] + b;
    }
  } else {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = a[k] + b;
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  out[threadIdx.x] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  std::vector<double2> tw(1024);
  for (int k = 0; k < 32; ++k)
    for (int l = 0; l < 32; ++l) {
      const double a = -2.0 * M_PI * k * l / 1024.0;
      tw[k * 32 + l] = make_double2(cos(a), sin(a));
    }
  double2 *dtw, *dout;
  long long* dcyc;
  cudaMalloc(&dtw, 1024 * sizeof(double2));
  cudaMalloc(&dout, nsm * 1024 * sizeof(double2));
  cudaMalloc(&dcyc, sizeof(long long));
  cudaMemcpy(dtw, tw.data(), 1024 * sizeof(double2), cudaMemcpyHostToDevice);
  const size_t smem = (1024 + 8 * 32 * kX) * sizeof(double2);
  cudaFuncSetAttribute(kfft<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kfft<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kfft<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kfft<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[4] = {"warp_fft1024 (rec tw)", "warp_fft1024 (table tw)", "Dft<32> x1", "Dft<32> x2"};
  const int iters = 200;
  for (int mode = 0; mode < 4; ++mode) {
    for (int warps = 1; warps <= 8; warps *= 2) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(dcyc, 0, sizeof(long long));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        if (mode == 0) kfft<0><<<nsm, 32 * warps, smem>>>(dout, dtw, iters, dcyc);
        if (mode == 1) kfft<1><<<nsm, 32 * warps, smem>>>(dout, dtw, iters, dcyc);
        if (mode == 2) kfft<2><<<nsm, 32 * warps, smem>>>(dout, dtw, iters, dcyc);
        if (mode == 3) kfft<3><<<nsm, 32 * warps, smem>>>(dout, dtw, iters, dcyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        long long cyc = 0;
        cudaMemcpy(&cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
        if (rep == 1)
          printf("%-26s warps/SM %d: %7.1f cycles per warp-iteration, %7.1f cycles per item per SM  (%.3f ms)\n",
                 names[mode], warps, (double)cyc / iters, (double)cyc / iters / warps, ms);
      }
    }
  }
  double* dd;
  cudaMalloc(&dd, 1024 * sizeof(double));
  for (int ilp = 1; ilp <= 8; ilp *= 8) {
    for (int rep = 0; rep < 2; ++rep) {
      kdadd<<<1, 32>>>(dd, 1000, ilp, dcyc);
      long long cyc = 0;
      cudaMemcpy(&cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
      if (rep == 1) printf("DADD 1 warp, ilp %d: %.2f cycles per dependent-step instruction\n", ilp, (double)cyc / (1000 * 16));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
