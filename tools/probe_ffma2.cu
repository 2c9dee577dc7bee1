// probe_ffma2.cu — FP32 FMA issue-rate microbenchmark on B200 (sm_100a): FFMA with register /
// constant-bank weights vs the packed FFMA2 (fma.rn.f32x2).  Each thread runs NACC independent
// accumulator chains for ITER iterations; FMA/clk/SM = fmas / (elapsed_s * sm_clock * SMs).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#define NACC 8
#define ITER 4096

struct W8 { float w[8]; };

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}

// weights in registers (loaded from global: not foldable)
__global__ void k_ffma_reg(const float* __restrict__ wg, float* out) {
  float w[8]; for (int i = 0; i < 8; i++) w[i] = wg[i];
  float x = out[threadIdx.x] + 1.f, a[NACC];
  for (int j = 0; j < NACC; j++) a[j] = x + j;
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
      for (int j = 0; j < NACC; j++) a[j] = __fmaf_rn(w[p], a[(j + 1) % NACC], a[j]);
  }
  float s = 0; for (int j = 0; j < NACC; j++) s += a[j];
  if (s == 12345.f) out[threadIdx.x] = s;
}
// weights as constant-bank operands (kernel parameter)
__global__ void k_ffma_const(W8 w, float* out) {
  float x = out[threadIdx.x] + 1.f, a[NACC];
  for (int j = 0; j < NACC; j++) a[j] = x + j;
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
      for (int j = 0; j < NACC; j++) a[j] = __fmaf_rn(w.w[p], a[(j + 1) % NACC], a[j]);
  }
  float s = 0; for (int j = 0; j < NACC; j++) s += a[j];
  if (s == 12345.f) out[threadIdx.x] = s;
}
// packed: NACC/2... use NACC pairs = 2*NACC fmas per p-step
__global__ void k_ffma2_reg(const float* __restrict__ wg, float* out) {
  unsigned long long w[8]; for (int i = 0; i < 8; i++) w[i] = pk(wg[i], wg[i]);
  float x = out[threadIdx.x] + 1.f; unsigned long long a[NACC];
  for (int j = 0; j < NACC; j++) a[j] = pk(x + j, x - j);
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
      for (int j = 0; j < NACC; j++) a[j] = f2(w[p], a[(j + 1) % NACC], a[j]);
  }
  unsigned long long s = 0; for (int j = 0; j < NACC; j++) s ^= a[j];
  if (s == 12345ull) out[threadIdx.x] = (float)s;
}
__global__ void k_ffma2_const(W8 wv, float* out) {
  float x = out[threadIdx.x] + 1.f; unsigned long long a[NACC];
  for (int j = 0; j < NACC; j++) a[j] = pk(x + j, x - j);
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
      for (int j = 0; j < NACC; j++) a[j] = f2(pk(wv.w[p], wv.w[p]), a[(j + 1) % NACC], a[j]);
  }
  unsigned long long s = 0; for (int j = 0; j < NACC; j++) s ^= a[j];
  if (s == 12345ull) out[threadIdx.x] = (float)s;
}
struct W8x2 { float2 w[8]; };
__global__ void k_ffma2_constpair(W8x2 wv, float* out) {
  float x = out[threadIdx.x] + 1.f; unsigned long long a[NACC];
  for (int j = 0; j < NACC; j++) a[j] = pk(x + j, x - j);
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
      for (int j = 0; j < NACC; j++) a[j] = f2(pk(wv.w[p].x, wv.w[p].y), a[(j + 1) % NACC], a[j]);
  }
  unsigned long long s = 0; for (int j = 0; j < NACC; j++) s ^= a[j];
  if (s == 12345ull) out[threadIdx.x] = (float)s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz (max)
  float *wg, *out;
  cudaMalloc(&wg, 64); cudaMalloc(&out, 1 << 20);
  float h[8]; for (int i = 0; i < 8; i++) h[i] = 0.5f + 0.01f * i;
  cudaMemcpy(wg, h, 32, cudaMemcpyHostToDevice);
  cudaMemset(out, 0, 1 << 20);
  W8 w; W8x2 w2; for (int i = 0; i < 8; i++) { w.w[i] = h[i]; w2.w[i] = make_float2(h[i], h[i]); }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    const int blocks = sms * (2048 / threads);
    for (int v = 0; v < 5; v++) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        if (v == 0) k_ffma_reg<<<blocks, threads>>>(wg, out);
        if (v == 1) k_ffma_const<<<blocks, threads>>>(w, out);
        if (v == 2) k_ffma2_reg<<<blocks, threads>>>(wg, out);
        if (v == 3) k_ffma2_const<<<blocks, threads>>>(w, out);
        if (v == 4) k_ffma2_constpair<<<blocks, threads>>>(w2, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      const double fmas = (double)blocks * threads * ITER * 8 * NACC * (v >= 2 ? 2 : 1);
      const char* nm[] = {"FFMA reg w", "FFMA const w", "FFMA2 reg w", "FFMA2 const w(pk)", "FFMA2 const pair"};
      printf("threads/CTA %4d  %-18s  %.3f ms  %.2f TFMA/s  %.1f FMA/clk/SM @max clk %d MHz\n", threads, nm[v], best,
             fmas / best / 1e9, fmas / (best * 1e-3) / (clk * 1e3) / sms, clk / 1000);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
