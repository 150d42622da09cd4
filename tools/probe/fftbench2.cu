// Microbenchmark: 1024-point fp64 FFT by a team of 64 threads (16 points each, two shared-memory
// exchanges: 16 x 16 x 4) against the warp-synchronous 32 x 32 transform (32 points per lane).
// Both with data in registers, repeated in place; checked against a direct DFT once.
#include <cmath>
#include <cstdio>
#include <vector>
#include "../../paper_2407_16559_b200/csrc/fft.cuh"
using namespace agk;

constexpr int kA1 = 68;              // exchange-1 row stride (16 rows x 64 + pad)
constexpr int kB2 = 21, kB1 = 84;    // exchange-2 strides: [k1][s][a + a/4]
constexpr int kTeamSm = 16 * kB1;    // double2 entries per team (>= 16 * kA1)

// x[t + 64 r] in v[r] (t = team thread 0..63) -> X[k1 + 16 (4 s' + i) + 256 b] in v[4 i + b]
// for thread (k1, s') = (t >> 2, t & 3). tw1: W_1024^{t k1} table [k1][t] (16 x 64);
// tw2: W_64^e, e < 64.
template <int SIGN>
__device__ __forceinline__ void team_fft1024(double2 (&v)[16], double2* sm, const double2* tw1, const double2* tw2,
                                             int t) {
  Dft<16, SIGN>::run(v);
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) {
    const double2 w = tw1[k1 * 64 + t];
    v[k1] = cmul(v[k1], SIGN < 0 ? w : cconj(w));
  }
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) sm[k1 * kA1 + t] = v[k1];
  asm volatile("bar.sync %0, 64;" ::"r"(1 + (threadIdx.x >> 6)) : "memory");
  const int k1 = t >> 2, s = t & 3;
#pragma unroll
  for (int u = 0; u < 16; ++u) v[u] = sm[k1 * kA1 + s + 4 * u];
  Dft<16, SIGN>::run(v);  // over u -> a
#pragma unroll
  for (int a = 1; a < 16; ++a) {
    const double2 w = tw2[s * a];
    v[a] = cmul(v[a], SIGN < 0 ? w : cconj(w));
  }
  asm volatile("bar.sync %0, 64;" ::"r"(1 + (threadIdx.x >> 6)) : "memory");
#pragma unroll
  for (int a = 0; a < 16; ++a) sm[k1 * kB1 + s * kB2 + a + (a >> 2)] = v[a];
  asm volatile("bar.sync %0, 64;" ::"r"(1 + (threadIdx.x >> 6)) : "memory");
  // thread (k1, s'): a = 4 s' + i, all four s -> DFT4 over s
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double2 q[4];
    const int a = 4 * s + i;
#pragma unroll
    for (int ss = 0; ss < 4; ++ss) q[ss] = sm[k1 * kB1 + ss * kB2 + a + (a >> 2)];
    Dft<4, SIGN>::run(q);
#pragma unroll
    for (int b = 0; b < 4; ++b) v[4 * i + b] = q[b];
  }
  asm volatile("bar.sync %0, 64;" ::"r"(1 + (threadIdx.x >> 6)) : "memory");
}

template <int TEAMS, int MINB>
__global__ void __launch_bounds__(TEAMS * 64, MINB) kteam(double2* out, const double2* g1, const double2* g2, int iters,
                                                          const double2* xin) {
  extern __shared__ double2 sm[];
  double2* tw1 = sm + TEAMS * kTeamSm;
  double2* tw2 = tw1 + 1024;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tw1[i] = g1[i];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) tw2[i] = g2[i];
  __syncthreads();
  const int team = threadIdx.x >> 6, t = threadIdx.x & 63;
  double2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = xin ? xin[t + 64 * r] : make_double2(t + r, r - t);
  for (int it = 0; it < iters; ++it) {
    team_fft1024<-1>(v, sm + team * kTeamSm, tw1, tw2, t);
    if (xin) break;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = make_double2(v[r].x * 1e-3, v[r].y * 1e-3);
  }
  const int k1 = t >> 2, s = t & 3;
  if (xin) {
    if (blockIdx.x == 0 && team == 0)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int b = 0; b < 4; ++b) out[k1 + 16 * (4 * s + i) + 256 * b] = v[4 * i + b];
    return;
  }
  double2 acc = czero();
#pragma unroll
  for (int r = 0; r < 16; ++r) acc = cadd(acc, v[r]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) kwarp(double2* out, const double2* gtw, int iters) {
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

static double2 wexp(double num, double den) {
  const long double a = -2.0L * 3.14159265358979323846264338327950288L * num / den;
  return make_double2((double)cosl(a), (double)sinl(a));
}

int main() {
  double2 *out, *g1, *g2, *gw, *xin;
  cudaMalloc(&out, 1 << 26);
  cudaMalloc(&g1, 1024 * 16);
  cudaMalloc(&g2, 64 * 16);
  cudaMalloc(&gw, 1024 * 16);
  cudaMalloc(&xin, 1024 * 16);
  std::vector<double2> h1(1024), h2(64), hw(1024), hx(1024), ho(1024);
  for (int k1 = 0; k1 < 16; ++k1)
    for (int t = 0; t < 64; ++t) h1[k1 * 64 + t] = wexp((double)k1 * t, 1024);
  for (int e = 0; e < 64; ++e) h2[e] = wexp(e, 64);
  for (int k = 0; k < 32; ++k)
    for (int l = 0; l < 32; ++l) hw[k * 32 + l] = wexp((double)l * k, 1024);
  for (int i = 0; i < 1024; ++i) hx[i] = make_double2(sin(0.37 * i) + 0.1, cos(0.11 * i * i));
  cudaMemcpy(g1, h1.data(), 1024 * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(g2, h2.data(), 64 * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(gw, hw.data(), 1024 * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(xin, hx.data(), 1024 * 16, cudaMemcpyHostToDevice);
  // correctness vs a long-double direct DFT
  {
    const size_t smem = (8 * kTeamSm + 1024 + 64) * sizeof(double2);
    cudaFuncSetAttribute(kteam<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kteam<8, 1><<<1, 512, smem>>>(out, g1, g2, 1, xin);
    cudaMemcpy(ho.data(), out, 1024 * 16, cudaMemcpyDeviceToHost);
    double maxe = 0, maxv = 0;
    for (int k = 0; k < 1024; ++k) {
      long double re = 0, im = 0;
      for (int n = 0; n < 1024; ++n) {
        const long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)((n * k) % 1024) / 1024;
        re += hx[n].x * cosl(a) - hx[n].y * sinl(a);
        im += hx[n].x * sinl(a) + hx[n].y * cosl(a);
      }
      maxe = fmax(maxe, fmax(fabs((double)(ho[k].x - re)), fabs((double)(ho[k].y - im))));
      maxv = fmax(maxv, fmax(fabs((double)re), fabs((double)im)));
    }
    printf("team fft rel err %.3e (%s)\n", maxe / maxv, cudaGetErrorString(cudaGetLastError()));
  }
  auto bench = [&](const char* name, auto launch, double ffts) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch(10);
    cudaEventRecord(a);
    launch(200);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-28s %.3f ms  %.1f Mfft/s  %s\n", name, ms, ffts * 200 / ms / 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  {
    const size_t smem = (8 * (kXS + 1) + 1024) * sizeof(double2);
    cudaFuncSetAttribute(kwarp<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bench("warp 32x32, 8 warps/SM", [&](int it) { kwarp<8, 1><<<148, 256, smem>>>(out, gw, it); }, 148.0 * 8);
  }
  {
    const size_t smem = (8 * kTeamSm + 1024 + 64) * sizeof(double2);
    cudaFuncSetAttribute(kteam<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bench("team 16x16x4, 16 warps/SM", [&](int it) { kteam<8, 1><<<148, 512, smem>>>(out, g1, g2, it, nullptr); },
          148.0 * 8);
  }
  {
    const size_t smem = (4 * kTeamSm + 1024 + 64) * sizeof(double2);
    cudaFuncSetAttribute(kteam<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bench("team, 2x8 warps/SM", [&](int it) { kteam<4, 2><<<296, 256, smem>>>(out, g1, g2, it, nullptr); }, 296.0 * 4);
  }
  {
    const size_t smem = (12 * kTeamSm + 1024 + 64) * sizeof(double2);
    cudaFuncSetAttribute(kteam<12, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bench("team, 24 warps/SM", [&](int it) { kteam<12, 1><<<148, 768, smem>>>(out, g1, g2, it, nullptr); },
          148.0 * 12);
  }
  return 0;
}
