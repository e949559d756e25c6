// tmem_rate.cu -- tcgen05.ld / tcgen05.st throughput (TMEM <-> registers) per SM on sm_100a.
// One CTA per SM, W warps (warp w reads lanes of quarter w % 4); each warp loads (or stores)
// 32 lanes x X columns x 4 bytes per instruction, `batch` instructions per wait.  Reports bytes per
// clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_rate tmem_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_1410_4984_b200/csrc/tc_util.cuh"

using namespace sgpx;

template <int MODE>  // 0 ld16 x2 per wait, 1 ld16 x1 per wait, 2 st16 x2 per wait, 3 ld8 x3 per wait
__global__ void rate(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  const uint32_t base = tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(32 * ((warp >> 2) & 7));
  float acc = 0.f;
  uint32_t r0[16], r1[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r0[i] = r1[i] = uint32_t(i + tid);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      tc::ld16(base, r0);
      tc::ld16(base + 16, r1);
      tc::ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += __uint_as_float(r0[i]) + __uint_as_float(r1[i]);
    } else if (MODE == 1) {
      tc::ld16(base, r0);
      tc::ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += __uint_as_float(r0[i]);
    } else if (MODE == 2) {
      tc::st16(base, r0);
      tc::st16(base + 16, r1);
      tc::st_wait();
      r0[it & 15] += 1u;
    } else {
      uint32_t a[8], b[8], c[8];
      tc::ld8(base, a);
      tc::ld8(base + 8, b);
      tc::ld8(base + 16, c);
      tc::ld_wait();
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += __uint_as_float(a[i]) + __uint_as_float(b[i]) + __uint_as_float(c[i]);
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) sink[tid] = acc;
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

template <int MODE>
void run(int warps, const char* name, double bytes_per_iter_per_warp) {
  const int iters = 4096, ctas = 148;
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, ctas * sizeof(unsigned long long));
  cudaMalloc(&sink, 1024 * sizeof(float));
  rate<MODE><<<ctas, 32 * warps>>>(iters, d, sink);
  rate<MODE><<<ctas, 32 * warps>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = bytes_per_iter_per_warp * warps * iters;
  printf("%-22s warps %2d: %8.1f clk/iter  %7.1f B/clk/SM\n", name, warps, mx / iters, bytes / mx);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 12, 16}) {
    run<0>(w, "ld16 x2 / wait", 2 * 32 * 16 * 4);
    run<1>(w, "ld16 x1 / wait", 32 * 16 * 4);
    run<3>(w, "ld8 x3 / wait", 3 * 32 * 8 * 4);
    run<2>(w, "st16 x2 / wait", 2 * 32 * 16 * 4);
  }
  return 0;
}
