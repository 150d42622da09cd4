// Hardware probe: fp64 FMA throughput, HBM copy, L2 write->read reuse, conditional graph nodes.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s at %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;i++){
    x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b);
    x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<n; i+=(size_t)gridDim.x*blockDim.x) b[i]=a[i];
}
__global__ void write_kernel(double2* b, size_t n, double v) {
  for (size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<n; i+=(size_t)gridDim.x*blockDim.x) b[i]=make_double2(v,i);
}
__global__ void read_kernel(const double2* __restrict__ b, size_t n, double* out) {
  double s=0;
  for (size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<n; i+=(size_t)gridDim.x*blockDim.x) s+=b[i].x;
  if (s==12345.0) out[0]=s;
}
__global__ void cond_body(int* counter, cudaGraphConditionalHandle h) {
  int c = ++(*counter);
  cudaGraphSetConditional(h, c < 1000 ? 1 : 0);
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("dev %s sms %d l2 %d MB persistL2max %d MB smemOptin %zu clock %d\n", p.name, p.multiProcessorCount, p.l2CacheSize>>20, p.persistingL2CacheMaxSize>>20, p.sharedMemPerBlockOptin, p.clockRate);
  double* out; CK(cudaMalloc(&out, 148*8*1024*8));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int iters=20000;
  for (int rep=0;rep<3;rep++){
  cudaEventRecord(e0); dfma_kernel<<<148*8,256>>>(out,iters,1.0000001,1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1);
  printf("dfma: %.2f TFLOP/s\n", 2.0*8*iters*148*8*256/(ms*1e-3)/1e12);}
  size_t big = (size_t)1<<27; // 2 GiB of double2
  double2 *a,*b; CK(cudaMalloc(&a,big*16)); CK(cudaMalloc(&b,big*16));
  write_kernel<<<148*8,512>>>(a,big,1.0); CK(cudaDeviceSynchronize());
  for (int rep=0;rep<3;rep++){
  cudaEventRecord(e0); copy_kernel<<<148*8,512>>>(a,b,big); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1); printf("copy 2GiB: %.1f GB/s\n", 2.0*big*16/(ms*1e-3)/1e9);}
  for (size_t mib : {8, 16, 32, 48, 64, 96, 128, 512}) {
    size_t n = mib*(1<<20)/16;
    for (int rep=0;rep<3;rep++){
    write_kernel<<<148*8,512>>>(b,big,2.0); // flush L2
    cudaEventRecord(e0); write_kernel<<<148*8,512>>>(a,n,1.0); read_kernel<<<148*8,512>>>(a,n,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); if(rep==2) printf("write+read %zu MiB: %.1f us -> %.1f GB/s eff\n", mib, ms*1e3, 2.0*n*16/(ms*1e-3)/1e9);}
  }
  // conditional while graph
  int* counter; CK(cudaMalloc(&counter,4)); CK(cudaMemset(counter,0,4));
  cudaGraph_t g; CK(cudaGraphCreate(&g,0));
  cudaGraphConditionalHandle h; CK(cudaGraphConditionalHandleCreate(&h,g,1,cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {}; cp.type=cudaGraphNodeTypeConditional; cp.conditional.handle=h; cp.conditional.type=cudaGraphCondTypeWhile; cp.conditional.size=1;
  cudaGraphNode_t cn; CK(cudaGraphAddNode(&cn,g,nullptr,0,&cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreate(&s);
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  cond_body<<<1,1,0,s>>>(counter,h);
  CK(cudaStreamEndCapture(s, nullptr));
  cudaGraphExec_t ge; CK(cudaGraphInstantiate(&ge,g,0));
  cudaEventRecord(e0,s); CK(cudaGraphLaunch(ge,s)); cudaEventRecord(e1,s); CK(cudaEventSynchronize(e1));
  int hc; cudaMemcpy(&hc,counter,4,cudaMemcpyDeviceToHost); cudaEventElapsedTime(&ms,e0,e1);
  printf("while graph: counter %d, %.2f us per iter\n", hc, ms*1e3/hc);
  return 0;
}
