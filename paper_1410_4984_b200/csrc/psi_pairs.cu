// psi_pairs.cu -- tensor-core forward psi2 (Phi) with inducing PAIRS as rows.
//
// Reference: psi_stats.hpp:221-277 (pair blocks: Phi_ab += sum_n c2_n pconst_ab exp(-e_nab)).
// With the translation and factorisation of DESIGN.md §3 every exponent is a bilinear form:
//
//   log2 v_nab = F_ab . H_n + B_n,
//   F_ab = [z_a o z_b, z_a + z_b, z_a^2 + z_b^2]            (3Q pair features, per evaluation)
//   H_n  = [K_n, al_n, be_n]                               (3Q datapoint features, per chunk)
//
// so a 128-pair x 256-datapoint tile is ONE tcgen05 MMA (kind::tf32, K = 3Q padded to 8, hi/lo
// split of both operands = 3 MMAs per K-step, ~fp32 accuracy), and Phi_ab is the row sum of
// ex2(D + B_n): each consumer thread owns one pair row, so there is no cross-lane reduction and
// an element costs one MUFU.EX2 + 2 FP32 instructions.
//
// CTA = 8 warps: warps 0-3 consume TMEM lanes 0..127 (pairs); warps 4-7 produce the datapoint
// features of the next chunk; lane 0 of warp 4 issues the MMAs.  TMEM: two 256-column D stages.
// Grid = (pair tiles) x (datapoint splits); CTA (rt, ns) writes its 128 fp64 row sums to
// phi_part[ns][pair] (single writer), reduced over ns in fixed order afterwards.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <atomic>

#include "psi_common.cuh"
#include "psi_kernels.cuh"
#include "tc_util.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;

namespace {
using namespace dev;

// CTA tile: kTiles pair tiles of 128 rows x kNC datapoints per chunk.  TMEM stage = kTiles * kNC
// = 256 columns, two stages = all 512 columns.  Warps: 4 * kTiles consumers (warp w reads TMEM
// lane quarter w & 3 of tile w >> 2; two consumer warps per SM sub-partition), then kNC / 32
// producers (one datapoint per thread per chunk); the first producer thread issues the MMAs.
constexpr int kTiles = 2;
constexpr int kNC = 128;                         // datapoints (MMA N) per chunk
constexpr int kRows = 128 * kTiles;              // pairs per CTA
constexpr int kConsumers = 128 * kTiles;         // consumer threads
constexpr int kProducers = kNC;                  // producer threads
constexpr int kThreads = kConsumers + kProducers;
constexpr int kStageCols = kTiles * kNC;         // TMEM columns per stage

__host__ __device__ constexpr int kdim_pairs(int q) { return (3 * q + 7) / 8 * 8; }

size_t pairs_smem_bytes(int q, int m, int qv) {
  const int K = kdim_pairs(q);
  const int mv = (m + 3) / 4 * 4;
  size_t f = 2 * size_t(kRows) * K           // A (pair features) hi/lo, kTiles tiles
             + 2 * 2 * size_t(kNC) * K       // B (datapoint features) hi/lo x 2 stages
             + 4 * kNC                       // B_n x 4-slot ring
             + size_t(mv) * qv;              // Zc
  return f * 4 + 16 * sizeof(uint64_t) + 64;
}

template <int Q>
__global__ void __launch_bounds__(kThreads, 1)
    psi2_fwd_pairs_kernel(PsiConst P, int64_t n_per_split, double* __restrict__ phi_part) {
  constexpr int K = (3 * Q + 7) / 8 * 8;
  constexpr int KS = K / 8;
  extern __shared__ __align__(1024) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = P.m, qv = P.qv;
  const int64_t npairs = int64_t(m) * (m + 1) / 2;
  float* A = sm;                          // [tile][hi|lo][128 x K]
  float* Bf = A + 2 * kRows * K;          // [stage][hi|lo][kNC x K]
  // B_n ring of 4 slots (slot c & 3): d_full(c-2) implies the issuer saw d_empty(c-4), so the
  // consumers are done with slot c & 3 when the producers rewrite it.
  float* Bn = Bf + 2 * 2 * kNC * K;       // [slot][kNC]
  float* Zc = Bn + 4 * kNC;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Zc + P.mv * qv);  // b_full[2], d_full[2], d_empty[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);
  uint64_t* b_full = bar;
  uint64_t* d_full = bar + 2;
  uint64_t* d_empty = bar + 4;

  for (int i = tid; i < P.mv * qv; i += blockDim.x) Zc[i] = P.zc[i];
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  if (tid == 0) {
    tc::mbar_init(&b_full[0], kProducers);
    tc::mbar_init(&b_full[1], kProducers);
    tc::mbar_init(&d_full[0], 1);
    tc::mbar_init(&d_full[1], 1);
    tc::mbar_init(&d_empty[0], kConsumers);
    tc::mbar_init(&d_empty[1], kConsumers);
    tc::mbar_fence_init();
  }
  __syncthreads();
  // pair features of this CTA's rows (p = kRows * blockIdx.x + r), hi/lo, canonical K-major
  const int64_t p0 = int64_t(blockIdx.x) * kRows;
  if (tid < kRows) {
    const int64_t p = p0 + tid;
    int a = 0, b = 0;
    if (p < npairs) {  // invert the m1-major upper-triangle index (psi_stats.hpp:85-97)
      int64_t rem = p;
      while (rem >= m - a) {
        rem -= m - a;
        ++a;
      }
      b = a + int(rem);
    }
    const bool vp = p < npairs;
    float* at = A + (tid >> 7) * 2 * 128 * K;
    const int r = tid & 127;
    for (int k = 0; k < K; k += 4) {
      float h[4], l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = k + u;
        float x = 0.f;
        if (vp && kk < 3 * Q && (kk % Q) < P.q) {
          const int q = kk % Q;
          const float za = Zc[a * qv + q], zb = Zc[b * qv + q];
          x = kk < Q ? za * zb : (kk < 2 * Q ? za + zb : fmaf(za, za, zb * zb));
        }
        h[u] = tc::tf32_hi(x);
        l[u] = x - h[u];
      }
      *reinterpret_cast<float4*>(at + tc::canon(r, k, K)) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(at + 128 * K + tc::canon(r, k, K)) = make_float4(l[0], l[1], l[2], l[3]);
    }
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t nb = int64_t(blockIdx.y) * n_per_split;
  const int64_t ne = min(P.n, nb + n_per_split);
  const int nchunks = int(nb < ne ? (ne - nb + kNC - 1) / kNC : 0);

  if (tid >= kConsumers) {
    // ---------------- producers: datapoint features of chunk c into stage c & 1 ----------------
    const int r = tid - kConsumers;  // datapoint row of the chunk
    const uint32_t idesc = tc::idesc_tf32(128, kNC);
    // raw inputs of the next chunk are prefetched into registers (all loads in flight at once:
    // one memory latency per chunk instead of one per load)
    double rm[Q], rs[Q];
    auto load_raw = [&](int c) {
      int64_t n = nb + int64_t(c) * kNC + r;
      n = n < ne ? n : nb;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int qq = q < P.q ? q : 0;
        rm[q] = __ldg(P.mu + qq * P.ld_mu + n);
        rs[q] = P.expected ? __ldg(P.s + qq * P.ld_s + n) : 0.0;
      }
    };
    if (nchunks > 0) load_raw(0);
    for (int c = 0; c < nchunks; ++c) {
      const int st = c & 1;
      float kk[Q], al[Q], be[Q];
      const bool valid = nb + int64_t(c) * kNC + r < ne;
      float bsum = valid ? 2.f * P.log2_var : -CUDART_INF_F;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        kk[q] = al[q] = be[q] = 0.f;
        if (q < P.q && valid) {
          // t = 1 + 2 S / l^2,  d2 = 1 / (2 S + l^2) = il2 / t  (MUFU.RCP / MUFU.LG2 forms)
          const float mu = float(rm[q] - P.center[q]);
          const float sv = float(rs[q]);
          const float il2 = P.il2[q];
          const float t = fmaf(2.f * sv, il2, 1.f);
          const float d2 = __fdividef(il2, t);
          const float a = kLog2e * d2 * mu;
          kk[q] = (kLog2e * il2) * sv * d2;
          al[q] = a;
          be[q] = -0.25f * kLog2e * (il2 + d2);
          bsum = fmaf(-0.5f, __log2f(t), fmaf(-a, mu, bsum));
        }
      }
      if (c + 1 < nchunks) load_raw(c + 1);
      if (c >= 2) tc::mbar_wait(&d_full[st], ((c - 2) >> 1) & 1);  // MMA(c-2) has read this stage
      float* bh = Bf + st * 2 * kNC * K;
      float* bl = bh + kNC * K;
      Bn[(c & 3) * kNC + r] = bsum;
#pragma unroll
      for (int k = 0; k < K; k += 4) {
        float hh[4], ll[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kx = k + u;
          const float x = kx < Q ? kk[kx % Q] : (kx < 2 * Q ? al[kx % Q] : (kx < 3 * Q ? be[kx % Q] : 0.f));
          hh[u] = tc::tf32_hi(x);
          ll[u] = x - hh[u];
        }
        *reinterpret_cast<float4*>(bh + tc::canon(r, k, K)) = make_float4(hh[0], hh[1], hh[2], hh[3]);
        *reinterpret_cast<float4*>(bl + tc::canon(r, k, K)) = make_float4(ll[0], ll[1], ll[2], ll[3]);
      }
      tc::fence_async_smem();
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&b_full[st])) : "memory");
      if (r == 0) {  // MMA issuer
        tc::mbar_wait(&b_full[st], (c >> 1) & 1);
        if (c >= 2) tc::mbar_wait(&d_empty[st], ((c - 2) >> 1) & 1);
        tc::fence_after();
        const uint64_t b_hi = tc::desc(tc::smem_u32(bh), K), b_lo = tc::desc(tc::smem_u32(bl), K);
#pragma unroll
        for (int tt = 0; tt < kTiles; ++tt) {
          const uint32_t d = tmem + st * kStageCols + tt * kNC;
          const float* at = A + tt * 2 * 128 * K;
          const uint64_t a_hi = tc::desc(tc::smem_u32(at), K), a_lo = tc::desc(tc::smem_u32(at + 128 * K), K);
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const uint64_t aa = (t == 2) ? a_lo : a_hi, bb = (t == 1) ? b_lo : b_hi;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) tc::mma_ss(d, aa + 16 * ks, bb + 16 * ks, idesc, (t | ks) ? 1u : 0u);
          }
        }
        tc::commit(&d_full[st]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- consumers: one pair row per thread ----------------
    const int tile = warp >> 2;
    const uint32_t lane_off = uint32_t(32 * (warp & 3)) << 16;
    double acc = 0.0;
    for (int c = 0; c < nchunks; ++c) {
      const int st = c & 1;
      tc::mbar_wait(&d_full[st], (c >> 1) & 1);
      tc::fence_after();
      const uint32_t d = tmem + st * kStageCols + tile * kNC + lane_off;
      const float* bn = Bn + (c & 3) * kNC;
      float s4[4] = {0.f, 0.f, 0.f, 0.f};  // four independent FADD chains
      uint32_t rr[32];
      tc::ld32(d, rr);
#pragma unroll 1
      for (int j = 0; j < kNC; j += 32) {
        tc::ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(rr[i]);
        if (j + 32 < kNC) tc::ld32(d + j + 32, rr);  // prefetch the next 32 columns
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 b4 = *reinterpret_cast<const float4*>(bn + j + i);
          s4[0] += ex2(v[i] + b4.x);
          s4[1] += ex2(v[i + 1] + b4.y);
          s4[2] += ex2(v[i + 2] + b4.z);
          s4[3] += ex2(v[i + 3] + b4.w);
        }
      }
      tc::ld_wait();
      acc += double((s4[0] + s4[1]) + (s4[2] + s4[3]));
      tc::fence_before();
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&d_empty[st])) : "memory");
    }
    const int64_t p = p0 + tid;
    if (p < npairs) phi_part[int64_t(blockIdx.y) * npairs + p] = acc;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// packed[4 + p] = sum_ns phi_part[ns][p]  (fixed order)
__global__ void phi_reduce_kernel(const double* __restrict__ phi_part, int ns, int64_t npairs,
                                  double* __restrict__ packed) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < npairs; p += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < ns; ++i) s += phi_part[i * npairs + p];
    packed[4 + p] = s;
  }
}

void pairs_grid(const PsiConst& P, int num_sms, int* rt, int* ns) {
  const int64_t npairs = int64_t(P.m) * (P.m + 1) / 2;
  *rt = int((npairs + kRows - 1) / kRows);
  const int64_t nchunks = (P.n + kNC - 1) / kNC;
  // splits of the datapoint range: fill whole waves of one CTA per SM
  int best = 1;
  double best_eff = -1.0;
  for (int s = 1; s <= 64 && (s <= nchunks || s == 1); ++s) {
    const int64_t ctas = int64_t(*rt) * s;
    const int64_t waves = (ctas + num_sms - 1) / num_sms;
    if (waves > 4) break;
    const double eff = double(ctas) / double(waves * num_sms);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  *ns = best;
}

template <int Q>
int launch_pairs_q(const PsiConst& P, double* phi_part, double* packed, int num_sms, cudaStream_t st) {
  int rt = 0, ns = 0;
  pairs_grid(P, num_sms, &rt, &ns);
  const size_t smem = pairs_smem_bytes(Q, P.m, P.qv);
  auto kern = psi2_fwd_pairs_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  const int64_t per = (P.n + ns - 1) / ns;
  const int64_t per_al = (per + kNC - 1) / kNC * kNC;
  kern<<<dim3(rt, ns), kThreads, smem, st>>>(P, per_al, phi_part);
  g_tc_launches.fetch_add(1);
  const int64_t npairs = int64_t(P.m) * (P.m + 1) / 2;
  phi_reduce_kernel<<<int((npairs + 255) / 256), 256, 0, st>>>(phi_part, ns, npairs, packed);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

bool pairs_supported(const PsiConst& P) {
  return P.q >= 1 && P.q <= 16 && pairs_smem_bytes(instantiated_q(P.q), P.m, P.qv) <= 227 * 1024;
}

int64_t pairs_part_doubles(const PsiConst& P, int num_sms) {
  int rt = 0, ns = 0;
  pairs_grid(P, num_sms, &rt, &ns);
  return int64_t(ns) * (int64_t(P.m) * (P.m + 1) / 2);
}

int psi2_forward_pairs(const PsiConst& P, double* phi_part, double* packed, int num_sms, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (instantiated_q(P.q)) {
    case 1: return launch_pairs_q<1>(P, phi_part, packed, num_sms, st);
    case 2: return launch_pairs_q<2>(P, phi_part, packed, num_sms, st);
    case 3: return launch_pairs_q<3>(P, phi_part, packed, num_sms, st);
    case 4: return launch_pairs_q<4>(P, phi_part, packed, num_sms, st);
    case 5: return launch_pairs_q<5>(P, phi_part, packed, num_sms, st);
    case 6: return launch_pairs_q<6>(P, phi_part, packed, num_sms, st);
    case 8: return launch_pairs_q<8>(P, phi_part, packed, num_sms, st);
    case 10: return launch_pairs_q<10>(P, phi_part, packed, num_sms, st);
    case 12: return launch_pairs_q<12>(P, phi_part, packed, num_sms, st);
    case 16: return launch_pairs_q<16>(P, phi_part, packed, num_sms, st);
    default: return 1;
  }
}

}  // namespace sgpx
