// Grid-barrier latency microbenchmark (B200): N back-to-back barriers of a cooperative grid of
// 148 CTAs x 512 threads; us per barrier for three orderings of the arrive / target / poll.
//   0: target from ctr[1] (relaxed load), then red.release, then acquire polls (library before r02)
//   1: red.release first, then the ctr[1] load and the first acquire poll in flight together
//   2: base cached in a register (no ctr[1] load per barrier)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2204_02064_b200/csrc -o gbar gbar.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"

using namespace perks;

// K distributed counters, 64 words (256 B) apart: CTA i arrives on counter i % K; pollers load all
// K and compare the sum
template <int K>
__global__ void __launch_bounds__(512, 1) kdist(unsigned *ctr, int iters, float *sink) {
  float acc = threadIdx.x;
  for (int n = 1; n <= iters; n++) {
    acc = acc * 1.0001f + 1.0f;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = n * gridDim.x;
      red_release_gpu(ctr + 64 * (blockIdx.x % K), 1u);
      while (true) {
        unsigned v[K];
#pragma unroll
        for (int k = 0; k < K; k++) v[k] = ld_relaxed_gpu(ctr + 64 * k);
        unsigned sum = 0;
#pragma unroll
        for (int k = 0; k < K; k++) sum += v[k];
        if ((int)(sum - target) >= 0) break;
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
// lower bound (NOT a correct barrier for data): relaxed arrive, relaxed polls, no fences
__global__ void __launch_bounds__(512, 1) relaxed_only(unsigned *ctr, int iters, float *sink) {
  float acc = threadIdx.x;
  for (int n = 1; n <= iters; n++) {
    acc = acc * 1.0001f + 1.0f;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = n * gridDim.x;
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      while ((int)(ld_relaxed_gpu(ctr) - target) < 0) {}
    }
    __syncthreads();
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
// release arrive only (acquire side relaxed): the cost of the release fence
__global__ void __launch_bounds__(512, 1) release_only(unsigned *ctr, int iters, float *sink) {
  float acc = threadIdx.x;
  for (int n = 1; n <= iters; n++) {
    acc = acc * 1.0001f + 1.0f;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = n * gridDim.x;
      red_release_gpu(ctr, 1u);
      while ((int)(ld_relaxed_gpu(ctr) - target) < 0) {}
    }
    __syncthreads();
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
// K counters; the last arriver of each (atom.acq_rel return value) bumps the top counter, which
// everyone polls
template <int K>
__global__ void __launch_bounds__(512, 1) ktree(unsigned *ctr, int iters, float *sink) {
  float acc = threadIdx.x;
  const int g = blockIdx.x % K;
  const unsigned gsize = (gridDim.x - g + K - 1) / K;  // CTAs in group g
  for (int n = 1; n <= iters; n++) {
    acc = acc * 1.0001f + 1.0f;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr + 64 * (g + 1)) : "memory");
      if (old + 1 == n * gsize) red_release_gpu(ctr, 1u);
      const unsigned target = n * K;
      while ((int)(ld_relaxed_gpu(ctr) - target) < 0) {}
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(unsigned *ctr, int iters, float *sink) {
  float acc = threadIdx.x;
  unsigned base = 0;
  if (MODE == 2) base = ld_relaxed_gpu(ctr + 1);
  for (int n = 1; n <= iters; n++) {
    acc = acc * 1.0001f + 1.0f;  // a little work between barriers
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned target;
      if (MODE == 0) {
        target = ld_relaxed_gpu(ctr + 1) + n * gridDim.x;
        red_release_gpu(ctr, 1u);
        while ((int)(ld_acquire_gpu(ctr) - target) < 0) {}
      } else if (MODE == 1) {
        red_release_gpu(ctr, 1u);
        const unsigned b = ld_relaxed_gpu(ctr + 1);
        unsigned v = ld_acquire_gpu(ctr);
        target = b + n * gridDim.x;
        while ((int)(v - target) < 0) v = ld_acquire_gpu(ctr);
      } else if (MODE == 2) {
        target = base + n * gridDim.x;
        red_release_gpu(ctr, 1u);
        while ((int)(ld_acquire_gpu(ctr) - target) < 0) {}
      } else if (MODE == 3) {  // relaxed polls, one acquire fence after
        red_release_gpu(ctr, 1u);
        const unsigned b = ld_relaxed_gpu(ctr + 1);
        unsigned v = ld_relaxed_gpu(ctr);
        target = b + n * gridDim.x;
        while ((int)(v - target) < 0) v = ld_relaxed_gpu(ctr);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else {  // cached base, relaxed polls, acquire fence
        target = base + n * gridDim.x;
        red_release_gpu(ctr, 1u);
        while ((int)(ld_relaxed_gpu(ctr) - target) < 0) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *ctr;
  float *sink;
  cudaMalloc(&ctr, 64 * 4 * 40);
  cudaMalloc(&sink, sizeof(float) * sms * 512);
  void *ks[4] = {(void *)kern<0>, (void *)relaxed_only, (void *)release_only, (void *)kern<4>};
  const char *names[4] = {"load-base, red, poll", "relaxed only (bound)", "release arrive, relaxed poll", "cached, relaxed polls, fence"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; rep++)
    for (int m = 0; m < 4; m++) {
      int iters = 20000;
      void *args[] = {&ctr, &iters, &sink};
      cudaMemset(ctr, 0, 64 * 4 * 40);
      cudaLaunchCooperativeKernel(ks[m], sms, 512, args, 0, 0);
      cudaMemset(ctr, 0, 64 * 4 * 40);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel(ks[m], sms, 512, args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%-28s %.3f us per barrier (%d CTAs)\n", names[m], ms * 1e3 / iters, sms);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
