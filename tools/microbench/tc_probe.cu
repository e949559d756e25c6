// tc_probe.cu -- unit probe of the hand-written tcgen05 path used by the psi kernels:
// TMEM alloc, SWIZZLE_NONE K-major smem descriptors, kind::tf32 MMA (M=128, N=32, K=16 as two
// K=8 steps), commit -> mbarrier, tcgen05.ld 32x32b.  Checks D = A B^T against fp64, once with
// plain TF32 operands and once with the 3xTF32 split (A_hi B_hi + A_hi B_lo + A_lo B_hi).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, N = 32, K = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// canonical K-major, no swizzle: core matrix = 8 rows x 16 B; LBO = stride between the two
// 16-byte k-chunks of one MMA (128 B here), SBO = stride between 8-row groups (K*32 B).
__device__ __forceinline__ int canon_off(int r, int k, int kdim) {  // in floats
  return (r >> 3) * (kdim * 8) + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

__global__ void probe(const float* A, const float* B, float* D, int split) {
  __shared__ __align__(1024) float sa[2][M * K];
  __shared__ __align__(1024) float sb[2][N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = A[i], h = split ? tf32_hi(x) : x;
    sa[0][canon_off(r, k, K)] = h;
    sa[1][canon_off(r, k, K)] = x - h;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = B[i], h = split ? tf32_hi(x) : x;
    sb[0][canon_off(r, k, K)] = h;
    sb[1][canon_off(r, k, K)] = x - h;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy smem writes -> visible to the MMA
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
  if (tid == 0) {
    int first = 1;
    const int terms = split ? 3 : 1;
    for (int t = 0; t < terms; ++t) {
      const int ai = (t == 2) ? 1 : 0, bi = (t == 1) ? 1 : 0;
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t da = make_desc(smem_u32(&sa[ai][0]) + ks * 256, 128, K * 32);
        const uint64_t db = make_desc(smem_u32(&sb[bi][0]) + ks * 256, 128, K * 32);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(first ? 0 : 1));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&mbar)));
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
  for (int j = 0; j < 32; ++j) D[row * N + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
  std::vector<float> a(M * K), b(N * K), d(M * N);
  uint64_t s = 12345;
  auto rnd = [&] {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return float((s >> 40) * (1.0 / (1ull << 24)) * 4.0 - 2.0);
  };
  for (auto& x : a) x = rnd();
  for (auto& x : b) x = rnd();
  float *dA, *dB, *dD;
  cudaMalloc(&dA, a.size() * 4);
  cudaMalloc(&dB, b.size() * 4);
  cudaMalloc(&dD, d.size() * 4);
  cudaMemcpy(dA, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  int bad = 0;
  for (int split = 0; split < 2; ++split) {
    probe<<<1, 128>>>(dA, dB, dD, split);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
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
    printf("split=%d max|err|=%.3e (max|ref| %.3f) rel %.3e  D[0][0]=%f D[127][31]=%f\n", split, maxerr, maxref,
           maxerr / maxref, d[0], d[M * N - 1]);
    if (maxerr / maxref > (split ? 1e-5 : 2e-3)) bad = 1;
  }
  printf(bad ? "TC PROBE FAIL\n" : "TC PROBE OK\n");
  return bad;
}
