// issue_cost.cu -- issue throughput of the MMA warp's bookkeeping instructions on sm_100a:
// tcgen05.commit (no wait), tcgen05.fence::after_thread_sync, mbarrier try_wait on a completed
// phase, and tcgen05.mma (kind::f16, A in TMEM, N = 96) back-to-back.  One warp per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_cost issue_cost.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_1410_4984_b200/csrc/tc_util.cuh"

using namespace sgpx;

template <int MODE>
__global__ void cost(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint32_t sm[];
  __shared__ __align__(8) uint64_t bar[9];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 16; i += blockDim.x) sm[i] = 0u;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  if (tid == 0) {
    for (int i = 0; i < 9; ++i) tc::mbar_init(&bar[i], 1);
    tc::mbar_fence_init();
  }
  asm volatile("fence.proxy.async.shared::cta;");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    if (MODE == 2) {  // complete phase 0 of bar[8] once
      if ((tid & 31) == 0) tc::mbar_arrive(&bar[8]);
      __syncwarp();
    }
    const uint32_t id = tc::idesc_f16(128, 96);
    const uint64_t b = tc::desc_sbo(tc::smem_u32(sm), 16 * 32);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE == 0) tc::commit_w(&bar[k]);
        else if (MODE == 1) tc::fence_after();
        else if (MODE == 2) tc::mbar_wait(&bar[8], 0);
        else if (MODE == 3) tc::mma_ts_f16_w(tmem, tmem + 256 + 8 * (k & 1), b, id, 1u);
        else if (MODE == 5) {  // per chunk: 6 MMA1 (f16 N=96) then 18 MMA3 (bf16 N=32), 3 commits
          if (k == 0) {
            const uint32_t id3 = tc::idesc_bf16(128, 32);
            for (int i = 0; i < 6; ++i) tc::mma_ts_f16_w(tmem, tmem + 256, b, id, 1u);
            for (int i = 0; i < 18; ++i) tc::mma_ts_f16_w(tmem + 128, tmem + 264, b, id3, 1u);
            tc::commit_w(&bar[0]);
            tc::commit_w(&bar[1]);
            tc::commit_w(&bar[2]);
          }
        } else if (MODE == 6) {  // same MMA count, all N=96
          if (k == 0) {
            for (int i = 0; i < 24; ++i) tc::mma_ts_f16_w(tmem, tmem + 256, b, id, 1u);
          }
        } else if (MODE == 7) {  // 18 MMA3 only (bf16 N=32)
          if (k == 0) {
            const uint32_t id3 = tc::idesc_bf16(128, 32);
            for (int i = 0; i < 18; ++i) tc::mma_ts_f16_w(tmem + 128, tmem + 264, b, id3, 1u);
          }
        } else if (MODE == 8) {  // alternate N=96 / N=32 every instruction
          if (k == 0) {
            const uint32_t id3 = tc::idesc_bf16(128, 32);
            for (int i = 0; i < 12; ++i) {
              tc::mma_ts_f16_w(tmem, tmem + 256, b, id, 1u);
              tc::mma_ts_f16_w(tmem + 128, tmem + 264, b, id3, 1u);
            }
          }
        } else {  // the kernel's per-chunk pattern: 6 MMA1 + 18 small MMA3 + 3 commits
          tc::mma_ts_f16_w(tmem, tmem + 256, b, id, 1u);
          if (k == 7) {
            tc::commit_w(&bar[0]);
            tc::commit_w(&bar[1]);
            tc::commit_w(&bar[2]);
          }
        }
      }
    }
    const long long t1 = clock64();
    tc::commit_w(&bar[8]);
    if ((tid & 31) == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    tc::mbar_wait(&bar[8], MODE == 2 ? 1 : 0);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

template <int MODE>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long));
  const int iters = 1000;
  cost<MODE><<<148, 32, 16384>>>(iters, d);
  cost<MODE><<<148, 32, 16384>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  unsigned long long h;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-40s %7.1f clk per instruction (issue loop)\n", name, double(h) / (iters * 8.0));
  cudaFree(d);
}

int main() {
  run<0>("tcgen05.commit (elect.sync)");
  run<1>("tcgen05.fence::after_thread_sync");
  run<2>("mbarrier try_wait, completed phase");
  run<3>("tcgen05.mma f16 ts N=96 K=16");
  run<4>("mma f16 ts N=96 + 3 commits / 8 mma");
  printf("per-chunk sequences (clk per 'instruction' below = per chunk / 8):\n");
  run<5>("6 x N96 f16 + 18 x N32 bf16 + 3 commits");
  run<6>("24 x N96 f16");
  run<7>("18 x N32 bf16");
  run<8>("12 x (N96 f16, N32 bf16) alternating");
  return 0;
}
