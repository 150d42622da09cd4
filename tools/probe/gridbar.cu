// Microbenchmark: software grid barrier (one 64-bit arrival counter, acquire spin) across a grid
// of co-resident CTAs, against chained empty launches (with and without programmatic dependent
// launch) — the latency budget of a persistent mid-size RHS kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridbar gridbar.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_bar(unsigned long long* cnt, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
    const unsigned long long target = (old / nb + 1) * nb;
    while (ld_acquire(cnt) < target) {
    }
  }
  __syncthreads();
}

__global__ void k_bar(unsigned long long* cnt, int iters, double* sink) {
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    grid_bar(cnt, gridDim.x);
    x = x * 1.0000001 + 1.0;
  }
  if (x == 12345.0) sink[0] = x;
}

__global__ void k_empty(int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
}

int main() {
  unsigned long long* cnt;
  double* sink;
  cudaMalloc(&cnt, 8);
  cudaMemset(cnt, 0, 8);
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int threads : {256, 512}) {
    for (int blocks : {74, 148, 296}) {
      if (threads == 512 && blocks == 296) continue;
      k_bar<<<blocks, threads>>>(cnt, 100, sink);
      cudaEventRecord(a);
      k_bar<<<blocks, threads>>>(cnt, 10000, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("grid barrier: %d CTAs x %d threads: %.3f us per barrier (%s)\n", blocks, threads, ms * 1e3 / 10000,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  // chained empty launches captured in a graph, with / without PDL
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int blocks : {1, 148}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < 300; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = blocks;
        cfg.blockDim = 256;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_empty, pdl);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(a, s);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("graph of empty launches: %d CTAs, pdl %d: %.3f us per launch (%s)\n", blocks, pdl, ms * 1e3 / 3000,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
