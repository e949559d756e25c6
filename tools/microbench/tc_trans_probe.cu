// tc_trans_probe.cu -- can a tile stored in the canonical K-major SWIZZLE_NONE layout (rows R,
// k = C) also serve as an MN-major B operand (N = C, K = R) of kind::tf32?  Tries both LBO/SBO
// assignments and reports the error of D = A * X (X[R][C]) against fp64.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, R = 32, C = 16;  // X: R x C;  D = A (M x R) * X  -> M x C

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ int canon(int r, int k, int kdim) {
  return (r >> 3) * (kdim * 8) + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void probe(const float* A, const float* X, float* D, uint32_t lbo, uint32_t sbo, int kstep_bytes) {
  __shared__ __align__(1024) float sa[M * R];
  __shared__ __align__(1024) float sx[R * C];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * R; i += blockDim.x) sa[canon(i / R, i % R, R)] = A[i];  // A K-major (k = R)
  for (int i = tid; i < R * C; i += blockDim.x) sx[canon(i / C, i % C, C)] = X[i];  // X stored K-major (rows R, k = C)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(32));
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
  // D f32, A/B tf32, A K-major, B MN-major (bit 16), N = C, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | (uint32_t(C >> 3) << 17) | (uint32_t(M >> 4) << 24);
  if (tid == 0) {
    for (int ks = 0; ks < R / 8; ++ks) {
      const uint64_t da = make_desc(smem_u32(sa) + ks * 256, 128, R * 32);
      const uint64_t db = make_desc(smem_u32(sx) + ks * kstep_bytes, lbo, sbo);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(ks ? 1 : 0));
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
  uint32_t r[16];
  const uint32_t taddr = tmem + (uint32_t(32 * warp) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int row = 32 * warp + lane;
  for (int j = 0; j < C; ++j) D[row * C + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
  std::vector<float> a(M * R), x(R * C), d(M * C);
  uint64_t s = 777;
  auto rnd = [&] {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    // values exactly representable in tf32 so the check is exact up to fp32 accumulation
    return float(int((s >> 40) % 2001) - 1000) / 256.0f;
  };
  for (auto& v : a) v = rnd();
  for (auto& v : x) v = rnd();
  float *dA, *dX, *dD;
  cudaMalloc(&dA, a.size() * 4);
  cudaMalloc(&dX, x.size() * 4);
  cudaMalloc(&dD, d.size() * 4);
  cudaMemcpy(dA, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  // candidates: (LBO, SBO, bytes per K-step of 8 rows)
  const uint32_t cands[][3] = {{128, C * 32, C * 32}, {C * 32, 128, C * 32}, {128, 256, C * 32}, {256, 128, C * 32}};
  int ok_any = 0;
  for (auto& cd : cands) {
    cudaMemset(dD, 0, d.size() * 4);
    probe<<<1, 128>>>(dA, dX, dD, cd[0], cd[1], int(cd[2]));
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("LBO=%u SBO=%u: CUDA error %s\n", cd[0], cd[1], cudaGetErrorString(e));
      return 2;
    }
    cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < C; ++j) {
        double ref = 0;
        for (int k = 0; k < R; ++k) ref += double(a[i * R + k]) * x[k * C + j];
        maxerr = std::fmax(maxerr, std::fabs(ref - d[i * C + j]));
        maxref = std::fmax(maxref, std::fabs(ref));
      }
    double r00 = 0;
    for (int k = 0; k < R; ++k) r00 += double(a[k]) * x[k * C];
    printf("  D[0][0]=%g ref %g  D[5][3]=%g\n", d[0], r00, d[5 * C + 3]);
    printf("LBO=%4u SBO=%4u kstep=%4u: max|err| %.3e (max|ref| %.1f)%s\n", cd[0], cd[1], cd[2], maxerr, maxref,
           maxerr / maxref < 1e-6 ? "  <-- OK" : "");
    if (maxerr / maxref < 1e-6) ok_any = 1;
  }
  printf(ok_any ? "TRANS PROBE OK\n" : "TRANS PROBE FAIL\n");
  return ok_any ? 0 : 1;
}
