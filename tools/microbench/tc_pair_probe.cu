// tc_pair_probe.cu -- CTA-pair (cta_group::2) tcgen05 semantics on sm_100a:
//   cluster (2,1,1); each CTA holds 128 rows of A (smem, or TMEM for the ts variant) and N/2 rows
//   of B (smem, same offset in both CTAs); the leader issues tcgen05.mma.cta_group::2 (M = 256);
//   the commit is multicast to both CTAs' mbarriers; each CTA reads its 128 x N block of D from
//   its own TMEM.  Also checks a remote mbarrier arrive (peer -> leader) through mapa.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int K = 16, N = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ int canon(int r, int k, int kdim) {
  return (r >> 3) * (kdim * 8) + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) probe(const float* A, const float* B, float* D, int ts) {
  __shared__ __align__(1024) float sa[128 * K];
  __shared__ __align__(1024) float sb[(N / 2) * K];
  __shared__ __align__(8) uint64_t mbar, peer_bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  for (int i = tid; i < 128 * K; i += blockDim.x) sa[canon(i / K, i % K, K)] = A[(rank * 128 + i / K) * K + i % K];
  for (int i = tid; i < (N / 2) * K; i += blockDim.x)
    sb[canon(i / K, i % K, K)] = B[(rank * (N / 2) + i / K) * K + i % K];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&peer_bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (ts) {  // A into TMEM columns [32, 48): thread = row of this CTA's half
    const int row = 32 * warp + lane;
    uint32_t r[16];
    for (int k = 0; k < 16; ++k) r[k] = __float_as_uint(A[(rank * 128 + row) * K + k]);
    const uint32_t ta = tmem + 32 + (uint32_t(32 * warp) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  // peer -> leader remote arrive: the leader waits for it before issuing (models "peer data ready")
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (rank == 1 && tid == 0) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&peer_bar)), "r"(0));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
  }
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
  if (rank == 0 && tid == 0) {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&peer_bar)), "r"(0));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t db = make_desc(smem_u32(sb) + ks * 256, 128, K * 32);
      if (ts) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
            "r"(tmem + 32 + ks * 8), "l"(db), "r"(idesc), "r"(ks ? 1 : 0));
      } else {
        const uint64_t da = make_desc(smem_u32(sa) + ks * 256, 128, K * 32);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(ks ? 1 : 0));
      }
    }
    const uint16_t mask = 3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&mbar)),
        "h"(mask));
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
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
  const int row = rank * 128 + 32 * warp + lane;
  for (int j = 0; j < N; ++j) D[row * N + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  const int M = 256;
  std::vector<float> a(M * K), b(N * K), d(M * N);
  uint64_t s = 5;
  auto rnd = [&] {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return float(int((s >> 40) % 2001) - 1000) / 256.0f;
  };
  for (auto& v : a) v = rnd();
  for (auto& v : b) v = rnd();
  float *dA, *dB, *dD;
  cudaMalloc(&dA, a.size() * 4);
  cudaMalloc(&dB, b.size() * 4);
  cudaMalloc(&dD, d.size() * 4);
  cudaMemcpy(dA, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  int ok = 1;
  for (int ts = 0; ts < 2; ++ts) {
    cudaMemset(dD, 0, d.size() * 4);
    probe<<<2, 128>>>(dA, dB, dD, ts);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("ts=%d CUDA error %s\n", ts, cudaGetErrorString(e));
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
    printf("cta_group::2 %s: max|err| %.3e (max|ref| %.1f) D[0][0]=%g D[200][20]=%g\n", ts ? "A=tmem" : "A=smem", maxerr,
           maxref, d[0], d[200 * N + 20]);
    if (maxerr / maxref > 1e-6) ok = 0;
  }
  printf(ok ? "PAIR PROBE OK\n" : "PAIR PROBE FAIL\n");
  return ok ? 0 : 1;
}
