// Do MUFU.EX2 and F2FP (cvt.rn.bf16x2.f32) share a pipe on sm_100a?  Throughput of each alone and interleaved.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned pk(float a, float b) { unsigned r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float x[8]; unsigned acc = 0; float s = 0;
  for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE & 1) x[i] = ex2f(x[i]) - 1.0f;
      if (MODE & 2) acc ^= pk(x[i], x[(i + 1) & 7] + 0.5f);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + float(acc);
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 1 << 22); cudaMallocManaged(&cyc, 8);
  const int iters = 2048, thr = 1024;
  auto run = [&](auto kern, const char* name, double ops_per_it) {
    kern<<<1, thr>>>(out, iters, cyc); cudaDeviceSynchronize();
    kern<<<1, thr>>>(out, iters, cyc); cudaDeviceSynchronize();
    printf("%-12s %8lld cycles  %.2f warp-instr/clk/SM\n", name, *cyc, ops_per_it * iters * (thr / 32) / double(*cyc));
  };
  run(k<1>, "ex2 only", 8);
  run(k<2>, "f2fp only", 8);
  run(k<3>, "both", 16);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
