// commit_lat.cu -- latency of tcgen05.commit -> mbarrier completion seen by the committing warp,
// with 0 or k queued MMAs (M = 128, N = 96, K = 8 tf32), and of a plain mbarrier arrive -> wait
// hand-off between two warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o commit_lat commit_lat.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_1410_4984_b200/csrc/tc_util.cuh"

using namespace sgpx;

__global__ void lat(int nmma, int ncommit, int iters, unsigned long long* out) {
  __shared__ __align__(8) uint64_t cb[8];
  extern __shared__ __align__(1024) float sm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 8 + 96 * 8; i += blockDim.x) sm[i] = 0.f;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    for (int k = 0; k < 8; ++k) tc::mbar_init(&cb[k], 1);
    tc::mbar_fence_init();
  }
  asm volatile("fence.proxy.async.shared::cta;");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t id = tc::idesc_tf32(128, 96);
    const uint64_t a = tc::desc(tc::smem_u32(sm), 8), b = tc::desc(tc::smem_u32(sm + 128 * 8), 8);
    uint32_t ph = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < nmma; ++k) tc::mma_ss_w(tmem, a, b, id, k ? 1u : 0u);
      for (int k = 0; k < ncommit - 1; ++k) tc::commit_w(&cb[k]);
      tc::commit_w(&bar[0]);
      tc::mbar_wait(&bar[0], ph);
      ph ^= 1u;
    }
    const unsigned long long t1 = clock64();
    if ((tid & 31) == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  } else if (warp == 1 || warp == 2) {
    // ping-pong between warps 1 and 2 over bar[1] (plain arrive / wait)
    __shared__ __align__(8) uint64_t pp[2];
    if (tid == 32) {
      tc::mbar_init(&pp[0], 1);
      tc::mbar_init(&pp[1], 1);
      tc::mbar_fence_init();
    }
    asm volatile("bar.sync 1, 64;");
    uint32_t ph = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (warp == 1) {
        if ((tid & 31) == 0) tc::mbar_arrive(&pp[0]);
        tc::mbar_wait(&pp[1], ph);
      } else {
        tc::mbar_wait(&pp[0], ph);
        if ((tid & 31) == 0) tc::mbar_arrive(&pp[1]);
      }
      ph ^= 1u;
    }
    const unsigned long long t1 = clock64();
    if (tid == 32 && blockIdx.x == 0) out[1] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 2 * sizeof(unsigned long long));
  const int iters = 2000;
  for (int nc : {1, 2, 3, 6})
  for (int nmma : {0, 1, 4, 9}) {
    lat<<<1, 96, 16384>>>(nmma, nc, iters, d);
    lat<<<148, 96, 16384>>>(nmma, nc, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    unsigned long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("commits %d ", nc);
    printf("mma %2d + commit + wait: %7.1f clk/iter   (warp ping-pong round trip %6.1f clk)\n", nmma,
           double(h[0]) / iters, double(h[1]) / iters);
  }
  return 0;
}
