// mma_rate2.cu -- tcgen05.mma issue rate for the shapes the row-tile kernel uses (and fp16
// alternatives): one CTA per SM, one warp issues a dependent chain of MMAs (accumulate into one
// D, as the kernel does) and reports clocks per instruction and MACs per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate2 mma_rate2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_1410_4984_b200/csrc/tc_util.cuh"

using namespace sgpx;

// KIND: 0 tf32 ss, 1 f16 ss, 2 bf16 ts, 3 tf32 ts
template <int KIND>
__global__ void rate(int n, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 16 + 256 * 16; i += blockDim.x) sm[i] = 0.f;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  asm volatile("fence.proxy.async.shared::cta;");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    uint32_t id;
    if (KIND == 0 || KIND == 3) id = tc::idesc_tf32(128, n);
    else if (KIND == 1) id = (1u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);  // f16 x f16
    else id = tc::idesc_bf16(128, n);
    const uint64_t a = tc::desc(tc::smem_u32(sm), 16), b = tc::desc(tc::smem_u32(sm + 128 * 16), 16);
    const uint32_t d = tmem, at = tmem + 256;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (KIND == 0) tc::mma_ss_w(d, a, b, id, 1u);
        else if (KIND == 1)
          asm volatile(
              "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(a), "l"(b), "r"(id), "r"(1u));
        else if (KIND == 2) tc::mma_ts_f16_w(d, at, b, id, 1u);
        else tc::mma_ts_w(d, at, b, id, 1u);
      }
    }
    tc::commit_w(&bar);
    tc::mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

template <int KIND>
void run(const char* name, int n, int kdim) {
  const int iters = 256, ctas = 148;
  unsigned long long* d;
  cudaMalloc(&d, ctas * sizeof(unsigned long long));
  rate<KIND><<<ctas, 32, 64 * 1024>>>(n, iters, d);
  cudaFuncSetAttribute(rate<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  rate<KIND><<<ctas, 32, 64 * 1024>>>(n, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
  const double per = mx / (iters * 16.0);
  printf("%-12s N=%3d K=%2d: %6.1f clk/MMA  %6.0f MAC/clk/SM\n", name, n, kdim, per, 128.0 * n * kdim / per);
  cudaFree(d);
}

int main() {
  for (int n : {32, 64, 96, 128, 192, 256}) run<0>("tf32 ss", n, 8);
  for (int n : {32, 64, 96, 128, 192, 256}) run<1>("f16 ss", n, 16);
  for (int n : {32, 64, 96, 128}) run<2>("bf16 ts", n, 16);
  for (int n : {32, 64, 96, 128}) run<3>("tf32 ts", n, 8);
  return 0;
}
