// FP32 FMA issue-rate microbenchmark (B200, sm_100a): which FFMA operand forms reach 128 FMA/clk/SM?
//   mode 0: FFMA R, R, UR, R  (weight a kernel parameter -> uniform register / constant)
//   mode 1: FFMA R, R, R, R   (weight in a per-thread register: 3 register sources)
//   mode 2: fma.rn.f32x2       (packed pairs, weight pair in registers)
//   mode 3: fma.rn.f32x2       (packed pairs, weight pair from a kernel parameter)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_rate ffma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NACC = 16, ITERS = 2048;

__device__ __forceinline__ unsigned long long pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack(unsigned long long v, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int MODE>
__global__ void kern(float *out, float w0, float w1, float seed) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = seed + threadIdx.x * 1e-7f + i;
  float wa = w0, wb = w1;
  if (MODE == 1 || MODE == 2) {  // move the weights into per-thread registers
    wa = w0 + threadIdx.x * 1e-30f;
    wb = w1 + threadIdx.x * 1e-30f;
  }
  if (MODE <= 1) {
    float x = seed;
#pragma unroll 1
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = fmaf(acc[i], (i & 1) ? wa : wb, x);
    }
  } else if (MODE == 4) {  // acc += data * w, w broadcast (the stencil form), data pairs varying
    unsigned long long a2[NACC / 2], d2[NACC / 2];
#pragma unroll
    for (int i = 0; i < NACC / 2; i++) {
      a2[i] = pack(acc[2 * i], acc[2 * i + 1]);
      d2[i] = pack(acc[2 * i] * 0.5f, acc[2 * i + 1] * 0.25f);
    }
    const unsigned long long wb = pack(wa, wa);
#pragma unroll 1
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
      for (int i = 0; i < NACC / 2; i++) a2[i] = fma2(d2[i], wb, a2[i]);
    }
#pragma unroll
    for (int i = 0; i < NACC / 2; i++) unpack(a2[i], acc[2 * i], acc[2 * i + 1]);
  } else {
    unsigned long long a2[NACC / 2];
#pragma unroll
    for (int i = 0; i < NACC / 2; i++) a2[i] = pack(acc[2 * i], acc[2 * i + 1]);
    const unsigned long long w2 = pack(wa, wb), x2 = pack(seed, seed);
#pragma unroll 1
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
      for (int i = 0; i < NACC / 2; i++) a2[i] = fma2(a2[i], w2, x2);
    }
#pragma unroll
    for (int i = 0; i < NACC / 2; i++) unpack(a2[i], acc[2 * i], acc[2 * i + 1]);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int threads = 512, blocks = sms * 4;
  float *out;
  cudaMalloc(&out, sizeof(float) * threads * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void (*ks[5])(float *, float, float, float) = {kern<0>, kern<1>, kern<2>, kern<3>, kern<4>};
  const char *names[5] = {"FFMA R,R,UR,R", "FFMA R,R,R,R", "fma.f32x2 regs", "fma.f32x2 param", "fma.f32x2 bcast w"};
  for (int m = 0; m < 5; m++) {
    for (int rep = 0; rep < 3; rep++) ks[m]<<<blocks, threads>>>(out, 0.999f, 0.998f, 1e-3f);
    cudaEventRecord(e0);
    const int REP = 10;
    for (int rep = 0; rep < REP; rep++) ks[m]<<<blocks, threads>>>(out, 0.999f, 0.998f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)REP * blocks * threads * ITERS * NACC;
    const double per_clk_sm = fmas / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%-18s %8.3f ms  %.1f TFMA/s  %.1f FMA/clk/SM (at the %d MHz base attribute)\n", names[m], ms,
           fmas / (ms * 1e-3) / 1e12, per_clk_sm, clk / 1000);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
