// Day-1 B200 probe: device attributes, cooperative+cluster launch acceptance,
// grid-barrier latency, launch gap, L2-resident copy bandwidth. Not product code.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s at %s:%d -> %s\n",#x,__FILE__,__LINE__,cudaGetErrorString(e));}}while(0)

__device__ __forceinline__ void red_release(unsigned* p, unsigned v){ asm volatile("red.release.gpu.global.add.u32 [%0], %1;"::"l"(p),"r"(v):"memory"); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p){ unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];":"=r"(v):"l"(p):"memory"); return v; }

__global__ void barrier_kernel(unsigned* ctr, int iters, long long* out){
  long long t0 = clock64();
  unsigned target = 0;
  for (int i=0;i<iters;i++){
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x==0){ red_release(ctr,1); while(ld_acquire(ctr) < target){} }
    __syncthreads();
  }
  if (blockIdx.x==0 && threadIdx.x==0) out[0] = clock64()-t0;
}
__global__ void empty_kernel(){}
__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x, s=(size_t)gridDim.x*blockDim.x;
  for(;i<n;i+=s) b[i]=a[i];
}
__global__ void __cluster_dims__(2,1,1) cluster_kernel(int* o){ if(threadIdx.x==0) o[blockIdx.x]=1; }

int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  int l2=0, smo=0, coop=0, clk=0, memclk=0; 
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize,0);
  cudaDeviceGetAttribute(&smo, cudaDevAttrMaxSharedMemoryPerBlockOptin,0);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch,0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate,0);
  printf("name=%s sms=%d cc=%d.%d l2=%d smem_optin=%d smem_per_sm=%zu regs_per_sm=%d coop=%d clk_khz=%d totalmem=%zu persistL2max=%d\n",
    p.name,p.multiProcessorCount,p.major,p.minor,l2,smo,p.sharedMemPerMultiprocessor,p.regsPerMultiprocessor,coop,clk,p.totalGlobalMem,p.persistingL2CacheMaxSize);
  // cooperative + cluster attribute together
  { int* o; CK(cudaMalloc(&o, 4096*4));
    cudaLaunchConfig_t cfg{}; cfg.gridDim=dim3(148); cfg.blockDim=dim3(128); cfg.stream=0;
    cudaLaunchAttribute at[2]; at[0].id=cudaLaunchAttributeCooperative; at[0].val.cooperative=1;
    cfg.attrs=at; cfg.numAttrs=1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_kernel, o); printf("coop+static cluster(2): %s\n", cudaGetErrorString(e)); cudaDeviceSynchronize(); cudaGetLastError();
    int ncl=0; cudaLaunchConfig_t c2=cfg; cudaLaunchAttribute a2[1]; a2[0].id=cudaLaunchAttributeClusterDimension; a2[0].val.clusterDim.x=2;a2[0].val.clusterDim.y=1;a2[0].val.clusterDim.z=1; c2.attrs=a2;c2.numAttrs=1;
    e=cudaOccupancyMaxActiveClusters(&ncl,(void*)cluster_kernel,&c2); printf("max active clusters(2)=%d %s\n",ncl,cudaGetErrorString(e));
  }
  // grid barrier latency for grid sizes
  unsigned* ctr; long long* out; CK(cudaMalloc(&ctr,4)); CK(cudaMalloc(&out,8));
  for(int g: {1,16,74,148,296}){
    for(int bs: {256,1024}){
      if (g==296 && bs==1024) continue;
      CK(cudaMemset(ctr,0,4));
      int iters=2000;
      cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
      barrier_kernel<<<g,bs>>>(ctr,10,out); CK(cudaDeviceSynchronize()); CK(cudaMemset(ctr,0,4));
      cudaEventRecord(a); barrier_kernel<<<g,bs>>>(ctr,iters,out); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms,a,b); long long cyc; cudaMemcpy(&cyc,out,8,cudaMemcpyDeviceToHost);
      printf("barrier grid=%d bs=%d: %.3f us/barrier (%.0f cyc)\n",g,bs,ms*1000/iters,(double)cyc/iters);
    }
  }
  // launch gap
  { cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
    for(int i=0;i<100;i++) empty_kernel<<<148,256>>>();
    cudaDeviceSynchronize(); cudaEventRecord(a); for(int i=0;i<1000;i++) empty_kernel<<<148,256>>>(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); printf("empty launch back-to-back: %.3f us/launch\n",ms);
    cudaGraph_t gr; cudaGraphExec_t ge; cudaStream_t s; cudaStreamCreate(&s);
    cudaStreamBeginCapture(s,cudaStreamCaptureModeGlobal); for(int i=0;i<1000;i++) empty_kernel<<<148,256,0,s>>>(); cudaStreamEndCapture(s,&gr);
    cudaGraphInstantiate(&ge,gr,0); cudaGraphLaunch(ge,s); cudaStreamSynchronize(s);
    cudaEventRecord(a,s); cudaGraphLaunch(ge,s); cudaEventRecord(b,s); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); printf("empty launch in graph: %.3f us/launch\n",ms);
  }
  // copy bandwidth vs size (L2 resident vs HBM)
  for(size_t mb: {8,16,32,48,64,128,1024}){
    size_t n=mb*1024*1024/16; float4*a,*b; CK(cudaMalloc(&a,n*16)); CK(cudaMalloc(&b,n*16)); cudaMemset(a,0,n*16);
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for(int i=0;i<5;i++) copy_kernel<<<148*8,256>>>(a,b,n);
    int it=50; cudaEventRecord(e0); for(int i=0;i<it;i++) copy_kernel<<<148*8,256>>>(a,b,n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1); printf("copy %zu MiB: %.1f GB/s (rd+wr), %.2f us/iter\n",mb, 2.0*n*16*it/(ms*1e-3)/1e9, ms*1000/it);
    cudaFree(a); cudaFree(b);
  }
  return 0;
}
