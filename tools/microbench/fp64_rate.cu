// fp64 throughput on one SM: SIMT DFMA vs DMMA (mma.sync m8n8k4 f64).  nvcc -arch=sm_100a fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, long long* cyc) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void dmma_kernel(double* out, int iters, long long* cyc) {
  double acc[4][2];
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 8);
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    dfma_kernel<<<1, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    dfma_kernel<<<1, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    double ops = double(threads) * iters * 8;
    printf("SIMT DFMA  threads %4d: %.1f DFMA/clk/SM\n", threads, ops / *cyc);
    dmma_kernel<<<1, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    dmma_kernel<<<1, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    double fmas = double(threads / 32) * iters * 4 * 256;  // m8n8k4 = 256 FMA
    printf("DMMA m8n8k4 threads %4d: %.1f FMA/clk/SM\n", threads, fmas / *cyc);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
// ---- latencies (one warp, dependent chains) ----
__global__ void lat_kernel(double* out, int iters, long long* cyc) {
  double acc[2] = {threadIdx.x * 1e-3, 1.0}, a = 1.0000001, b = 0.9999999, x = 2.0 + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(acc[0]), "+d"(acc[1]) : "d"(a), "d"(b));
  long long t1 = clock64();
  double y = x;
  for (int it = 0; it < iters; ++it) y = fma(y, a, 1e-12);
  long long t2 = clock64();
  double z = x;
  for (int it = 0; it < iters; ++it) z = rsqrt(z) + 1.5;
  long long t3 = clock64();
  double w = x;
  for (int it = 0; it < iters; ++it) w = sqrt(w) + 1.5;
  long long t4 = clock64();
  double v = x;
  for (int it = 0; it < iters; ++it) v = 1.0 / v + 1.5;
  long long t5 = clock64();
  out[threadIdx.x] = acc[0] + acc[1] + y + z + w + v;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
}
struct LatMain {
  LatMain() {
    double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 64);
    const int it = 1000;
    lat_kernel<<<1, 32>>>(out, it, cyc); cudaDeviceSynchronize();
    lat_kernel<<<1, 32>>>(out, it, cyc); cudaDeviceSynchronize();
    printf("latency (cycles per dependent op): DMMA %.1f  DFMA %.1f  rsqrt+add %.1f  sqrt+add %.1f  rcp+add %.1f\n",
           double(cyc[0]) / it, double(cyc[1]) / it, double(cyc[2]) / it, double(cyc[3]) / it, double(cyc[4]) / it);
  }
};
static LatMain lat_main_runs_after_main_statics;
