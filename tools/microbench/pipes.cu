// Pipe-throughput microbenchmark for sm_100a: FFMA vs FFMA2 (fma.rn.f32x2) vs MUFU.EX2.
// Used once to choose the psi-statistics inner-loop instruction mix.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__device__ __forceinline__ unsigned long long f2(unsigned long long x, unsigned long long a, unsigned long long b) {
  unsigned long long r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(a), "l"(b)); return r;
}
__global__ void k_ffma2(float* out, float a, float b) {
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *(unsigned long long*)&av, B = *(unsigned long long*)&bv;
  unsigned long long x[8];
  for (int j = 0; j < 8; ++j) { float2 t = make_float2(threadIdx.x + j, threadIdx.x - j); x[j] = *(unsigned long long*)&t; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = f2(x[k], A, B);
    }
  }
  float s = 0; for (int k = 0; k < 8; ++k) { float2 t = *(float2*)&x[k]; s += t.x + t.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ex2(float* out, float a) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f, x4 = x0 + .4f, x5 = x0 + .5f, x6 = x0 + .6f, x7 = x0 + .7f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x3));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x4)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x5));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x6)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x7));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
// mixed: 8 FFMA per EX2 (ratio of the psi2 inner loop) to see if MUFU overlaps the FMA pipe
__global__ void k_mix(float* out, float a, float b) {
  float x[8], e[8];
  for (int k = 0; k < 8; ++k) { x[k] = threadIdx.x + k; e[k] = -1.f * k; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[k] = fmaf(x[k], a, b);
      float t; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(x[k] * 1e-30f)); e[k] += t;
    }
  }
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k] + e[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int thr : {256, 512, 1024}) {
    int blocks = sms * (2048 / thr);
    double lanes = (double)blocks * thr;
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); k_ffma<<<blocks, thr>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double ffma = lanes * ITERS * 32 / (ms * 1e-3);
      cudaEventRecord(e0); k_ffma2<<<blocks, thr>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms2; cudaEventElapsedTime(&ms2, e0, e1);
      double ffma2 = lanes * ITERS * 32 * 2 / (ms2 * 1e-3);
      cudaEventRecord(e0); k_ex2<<<blocks, thr>>>(out, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms3; cudaEventElapsedTime(&ms3, e0, e1);
      double ex2 = lanes * ITERS * 32 / (ms3 * 1e-3);
      cudaEventRecord(e0); k_mix<<<blocks, thr>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms4; cudaEventElapsedTime(&ms4, e0, e1);
      double mix_ffma = lanes * ITERS * 64 / (ms4 * 1e-3);
      printf("thr=%d rep=%d FFMA %.2f Tfma/s (%.1f TFLOP/s)  FFMA2 %.2f Tfma/s  EX2 %.3f T/s  MIX(8:1) %.2f Tfma/s  [sms=%d clk=%d MHz]\n",
             thr, rep, ffma / 1e12, 2 * ffma / 1e12, ffma2 / 1e12, ex2 / 1e12, mix_ffma / 1e12, sms, clk / 1000);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
