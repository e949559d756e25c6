// mma_rate.cu -- tcgen05 kind::tf32 issue/throughput vs N, A source (smem / TMEM) and number of
// independent accumulators (dependency chains).  One CTA per SM, one issuing thread; reports
// cycles per MMA (M = 128, K = 8 per instruction) and achieved FMA/clk/SM.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int CHAINS, int ATMEM>
__global__ void rate(int n_dim, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 8 + 256 * 8; i += blockDim.x) sm[i] = 0.001f * (i % 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n_dim >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t da = make_desc(smem_u32(sm), 128, 8 * 32);
    const uint64_t db = make_desc(smem_u32(sm + 128 * 8), 128, 8 * 32);
    const uint32_t a_t = tmem + 448;  // A operand columns in TMEM (8 cols)
    const unsigned long long t0 = clock64();
    uint32_t dd[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) dd[c] = tmem + uint32_t(c * n_dim);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 48; ++k) {
        const uint32_t d = dd[k % CHAINS];
        const uint32_t acc = 1u;
        if (ATMEM)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
              "r"(a_t), "l"(db), "r"(idesc), "r"(acc));
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = (128 * 8 + 256 * 8) * 4;
  cudaFuncSetAttribute(rate<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<4, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 400;
  printf("%-6s %-6s %-7s %12s %14s\n", "N", "A", "chains", "clk/MMA", "FMA/clk/SM");
  for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
    for (int n : {16, 32, 64, 96, 128, 256})
      for (int chains : {1, 2, 4}) {
        if (n * chains > 448) continue;
        if (chains == 1) (a_tmem ? rate<1, 1> : rate<1, 0>)<<<sms, 128, smem>>>(n, iters, d);
        if (chains == 2) (a_tmem ? rate<2, 1> : rate<2, 0>)<<<sms, 128, smem>>>(n, iters, d);
        if (chains == 4) (a_tmem ? rate<4, 1> : rate<4, 0>)<<<sms, 128, smem>>>(n, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        unsigned long long cyc;
        cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        const double per = double(cyc) / (48.0 * iters);
        printf("%-6d %-6s %-7d %12.1f %14.0f\n", n, a_tmem ? "tmem" : "smem", chains, per, 128.0 * n * 8 / per);
      }
  return 0;
}
