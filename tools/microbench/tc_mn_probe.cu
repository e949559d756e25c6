// tc_mn_probe.cu -- which MN-major B layouts does kind::tf32 accept?  D = A (128 x 32) * X (32 x 32),
// X stored MN-major (N contiguous) in SWIZZLE_NONE / SW32 / SW128 canonical forms.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, KD = 32, N = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ int canonK(int r, int k, int kdim) {
  return (r >> 3) * (kdim * 8) + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t ltype) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (uint64_t(ltype) << 61);
}
// byte offset of X(mn, k) for mode: 0 = none (T=4 wide atoms), 1 = SW32 (8 wide), 2 = SW128 (32 wide)
__device__ __forceinline__ uint32_t off_mn(int mode, int mn, int k, uint32_t lbo, uint32_t sbo) {
  const int W = mode == 0 ? 4 : (mode == 1 ? 8 : 32);  // atom width in elements
  const int j = mn / W, e = mn % W, r = k & 7, kg = k >> 3;
  uint32_t a;
  if (mode == 0) a = uint32_t(j) * sbo + uint32_t(kg) * lbo + uint32_t(r) * 16 + e * 4;
  else a = uint32_t(j) * lbo + uint32_t(kg) * sbo + uint32_t(r) * (W * 4) + e * 4;
  if (mode == 1) a ^= ((a >> 7) & 1) << 4;
  if (mode == 2) a ^= ((a >> 7) & 7) << 4;
  return a;
}

__global__ void probe(const float* A, const float* X, float* D, int mode, uint32_t lbo, uint32_t sbo, uint32_t kstep) {
  __shared__ __align__(1024) float sa[M * KD];
  __shared__ __align__(1024) float sx[4096];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * KD; i += blockDim.x) sa[canonK(i / KD, i % KD, KD)] = A[i];
  for (int i = tid; i < 4096; i += blockDim.x) sx[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < KD * N; i += blockDim.x) {
    const int k = i / N, mn = i % N;
    sx[off_mn(mode, mn, k, lbo, sbo) / 4] = X[i];
  }
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
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
  const uint32_t ltype = mode == 0 ? 0 : (mode == 1 ? 6 : 2);
  if (tid == 0) {
    for (int ks = 0; ks < KD / 8; ++ks) {
      const uint64_t da = make_desc(smem_u32(sa) + ks * 256, 128, KD * 32, 0);
      const uint64_t db = make_desc(smem_u32(sx) + ks * kstep, lbo, sbo, ltype);
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
  std::vector<float> a(M * KD), x(KD * N), d(M * N);
  uint64_t s = 4242;
  auto rnd = [&] {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
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
  struct Cand { int mode; uint32_t lbo, sbo, kstep; const char* name; };
  const Cand cands[] = {
      {0, 512, 128, 512, "none  LBO=K-grp SBO=MN-chunk"}, {0, 128, 512, 512, "none  swapped"},
      {0, 1024, 128, 1024, "none  LBO=1024"},
      {1, 256, 1024, 1024, "sw32  LBO=MN-atom SBO=K-grp"}, {1, 1024, 256, 1024, "sw32  swapped"},
      {2, 1024, 1024, 1024, "sw128 single atom"}, {2, 0, 1024, 1024, "sw128 lbo0"}};
  int ok_any = 0;
  for (auto& c : cands) {
    cudaMemset(dD, 0, d.size() * 4);
    probe<<<1, 128>>>(dA, dX, dD, c.mode, c.lbo, c.sbo, c.kstep);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: CUDA error %s\n", c.name, cudaGetErrorString(e));
      return 2;
    }
    cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0, maxd = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double ref = 0;
        for (int k = 0; k < KD; ++k) ref += double(a[i * KD + k]) * x[k * N + j];
        maxerr = std::fmax(maxerr, std::fabs(ref - d[i * N + j]));
        maxref = std::fmax(maxref, std::fabs(ref));
        maxd = std::fmax(maxd, std::fabs(d[i * N + j]));
      }
    const bool ok = maxerr / maxref < 1e-6;
    printf("%-30s: max|err| %.3e max|D| %.3e (max|ref| %.1f)%s\n", c.name, maxerr, maxd, maxref, ok ? "  <-- OK" : "");
    ok_any |= ok;
  }
  printf(ok_any ? "MN PROBE OK\n" : "MN PROBE FAIL\n");
  return ok_any ? 0 : 1;
}
