// Probe: does a kernel that contains tcgen05.alloc get a lower occupancy from the runtime?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(288, 2) k_plain(int *p) { if (p[0] == 12345) p[1] = 1; }
__global__ void __launch_bounds__(288, 2) k_tmem(int *p, int cols) {
  __shared__ unsigned slot;
  if (p[0] == 12345 && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&slot)), "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(slot), "r"(cols) : "memory");
  }
}
__global__ void __launch_bounds__(288, 2) k_tmem_run(int *p, int cols, unsigned long long *t) {
  __shared__ unsigned slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&slot)), "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  __syncthreads();
  unsigned smid; asm("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) { t[blockIdx.x] = ((unsigned long long)smid << 32) | slot; }
  long long c0 = clock64(); while (clock64() - c0 < 2000000) {}
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(slot), "r"(cols) : "memory");
}
int main() {
  size_t sm[] = {0, 40000, 100000, 110000};
  for (size_t s : sm) {
    int a = 0, b = 0, c = 0;
    cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k_tmem_run, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_plain, 288, s);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_tmem, 288, s);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_tmem_run, 288, s);
    printf("smem=%zu occ plain=%d tmem=%d tmem_run=%d\n", s, a, b, c);
  }
  // actual co-residency: 296 CTAs (non-cooperative), 256 cols each, record smid + tmem address
  int *p; unsigned long long *t;
  cudaMalloc(&p, 64); cudaMemset(p, 0, 64);
  cudaMalloc(&t, 296 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_tmem_run<<<296, 288, 100000>>>(p, 256, t);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[296]; cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
  int cnt[200] = {0}; int maxc = 0;
  for (int i = 0; i < 296; i++) { int s = h[i] >> 32; cnt[s]++; if (cnt[s] > maxc) maxc = cnt[s]; }
  printf("run: err=%s ms=%.3f (one CTA spin ~1ms) max CTAs/SM seen=%d addr0=%llx addr1=%llx\n", cudaGetErrorString(err), ms, maxc,
         h[0] & 0xffffffffull, h[1] & 0xffffffffull);
  // cooperative launch of 296
  void *args[] = {&p, (void *)nullptr, &t};
  int cols = 256; args[1] = &cols;
  err = cudaLaunchCooperativeKernel((void *)k_tmem_run, 296, 288, args, 100000, 0);
  printf("coop 296: %s\n", cudaGetErrorString(err));
  err = cudaDeviceSynchronize();
  printf("coop sync: %s\n", cudaGetErrorString(err));
  return 0;
}
