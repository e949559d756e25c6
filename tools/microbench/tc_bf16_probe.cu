// tc_bf16_probe.cu -- kind::f16 (bf16 inputs, f32 accumulate) with A in TMEM (bf16x2 packed per
// 32-bit column, written by tcgen05.st) and B in shared memory (canonical K-major, 8 bf16 per
// 16-byte core-matrix row).  D = A (128 x 16) * B^T (B: 32 x 16).  Checks both packing orders.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, K = 32, N = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void probe(const float* A, const float* B, float* D, int lo_first) {
  __shared__ __align__(1024) __nv_bfloat16 sb[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;  // B[n][k], canonical K-major bf16
    sb[(r >> 3) * (K * 8) + (k >> 3) * 64 + (r & 7) * 8 + (k & 7)] = __float2bfloat16_rn(B[i]);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(64));
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
  {  // A row -> TMEM columns [32, 48): 16 columns of bf16x2
    const int row = 32 * warp + lane;
    uint32_t r[16];
    for (int c = 0; c < 16; ++c) {
      const float e0 = A[row * K + 2 * c], e1 = A[row * K + 2 * c + 1];
      uint32_t d;
      if (lo_first) asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(e1), "f"(e0));  // lo = e0
      else asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(e0), "f"(e1));           // lo = e1
      r[c] = d;
    }
    const uint32_t ta = tmem + 32 + (uint32_t(32 * warp) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // kind::f16: D f32 (bit 4), A bf16 (1 << 7), B bf16 (1 << 10), K-major both
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
  if (tid == 0) {
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t db = make_desc(smem_u32(sb) + ks * 256, 128, K * 16);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
          "r"(tmem + 32 + ks * 8), "l"(db), "r"(idesc), "r"(ks ? 1 : 0));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[32];
  const uint32_t taddr = tmem + (uint32_t(32 * warp) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int row = 32 * warp + lane;
  for (int j = 0; j < N; ++j) D[row * N + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  std::vector<float> a(M * K), b(N * K), d(M * N);
  uint64_t s = 31;
  auto rnd = [&] {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return float(int((s >> 40) % 255) - 127) / 16.0f;  // exact in bf16
  };
  for (auto& v : a) v = rnd();
  for (auto& v : b) v = rnd();
  float *dA, *dB, *dD;
  cudaMalloc(&dA, a.size() * 4);
  cudaMalloc(&dB, b.size() * 4);
  cudaMalloc(&dD, d.size() * 4);
  cudaMemcpy(dA, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  int ok = 0;
  for (int lo_first = 0; lo_first < 2; ++lo_first) {
    probe<<<1, 128>>>(dA, dB, dD, lo_first);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      printf("CUDA error\n");
      return 2;
    }
    cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += double(a[i * K + k]) * b[j * K + k];
        maxerr = std::fmax(maxerr, std::fabs(ref - d[i * N + j]));
        maxref = std::fmax(maxref, std::fabs(ref));
      }
    printf("lo_first=%d max|err| %.3e (max|ref| %.1f)%s\n", lo_first, maxerr, maxref, maxerr / maxref < 1e-6 ? "  OK" : "");
    if (maxerr / maxref < 1e-6) ok = 1;
  }
  printf(ok ? "BF16 PROBE OK\n" : "BF16 PROBE FAIL\n");
  return ok ? 0 : 1;
}
