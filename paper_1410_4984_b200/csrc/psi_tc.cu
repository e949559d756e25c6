// psi_tc.cu -- tensor-core (tcgen05, 3xTF32) variants of the psi-statistics kernels.
//
// Same sums as psi_kernels.cu (reference: proj/include/sgp/psi_stats.hpp:108-326); the psi2
// cross term  sum_q K_nq z_aq z_bq  of every (n, a, b) exponent comes out of one MMA per row tile:
//
//   row tile  = 32 datapoints (lanes) x 4 inducing points a (warps of a pipeline) = 128 rows
//   MMA1      : D1[r, b] = A1[r, :] . B1[b, :],  A1[(n,a), q] = K_nq z_aq,  B1[b, q] = z_bq
//               (K = Q padded to 8; hi/lo split of both operands, 3 MMAs per K-step ~ fp32 accuracy)
//   SIMT      : s = D1 + L_na + L_nb;  v = ex2(s)   (one MUFU.EX2 per element -- the roofline)
//   forward   : Phi_ab += sum over the 32 lanes (warp reduce-scatter), fp64 RED into CTA partials
//   backward  : G = U_ab v written back to TMEM (hi/lo), MMA2 (A from TMEM):
//               D2[r, :] = G[r, :] . [1 | z_b1 .. z_bQ]  ->  R_na = sum_b G, S_naq = sum_b G z_bq
//
// Two independent 4-warp pipelines per CTA (each owns 128 TMEM columns per stage and its own
// operand buffers) so one pipeline's MMA latency hides behind the other's SIMT work.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "psi_common.cuh"
#include "psi_kernels.cuh"
#include "tc_util.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;
std::atomic<int64_t> g_tc_launches{0};

namespace {
using namespace dev;

constexpr int kPipes = 2;       // backward: TMEM 256 columns per pipeline
constexpr int kPipesF = 4;      // forward: TMEM 128 columns per pipeline
constexpr int kThreadsF = 128 * kPipesF;

// Per-phase cycle counters (only when P.prof != null): accumulated by lane 0 of each pipeline's
// first warp.  Slots: 0 prologue, 1 A1 build + barrier, 2 MMA1 wait, 3 element loop, 4 MMA2 issue,
// 5 MMA2 wait, 6 contraction, 7 epilogue, 8 tiles.
#define TCP_MARK(var) long long var = P.prof ? clock64() : 0
#define TCP_ADD(slot, from) \
  do { if (P.prof && wq == 0 && lane == 0) atomicAdd(P.prof + (slot), (unsigned long long)(clock64() - (from))); } while (0)
constexpr int kThreadsTC = 128 * kPipes;

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

struct TCLayout {
  int k1;    // MMA1 K (2Q rounded to 8)
  int n1;    // MMA1 N (M rounded to 16), <= 128
  int k2;    // MMA2 K (M rounded to 8)
  int n2;    // MMA2 N (Q+1 rounded to 16)
};

__host__ __device__ inline TCLayout tc_layout(int q, int m) {
  return TCLayout{round_up(2 * q, 8), round_up(m, 16), round_up(m, 8), round_up(q + 1, 16)};
}

// B1[b, :] = [z_b1..z_bQ, z_b1^2..z_bQ^2] (centred Z) as the K-major B operand, hi and lo planes.
__device__ __forceinline__ void build_b1(const PsiConst& P, const TCLayout& L, const float* Zc, float* b1) {
  const int tot = L.n1 * L.k1;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    const int b = i / L.k1, k = i - b * L.k1;
    float z = 0.f;
    if (b < P.m && k < 2 * P.q) {
      const float zz = Zc[b * P.qv + (k < P.q ? k : k - P.q)];
      z = k < P.q ? zz : zz * zz;
    }
    const float h = tc::tf32_hi(z);
    b1[tc::canon(b, k, L.k1)] = h;
    b1[L.n1 * L.k1 + tc::canon(b, k, L.k1)] = z - h;
  }
}

// A1 row of one tile, row r = 32*wq + lane <-> (datapoint lane, inducing a):
//   [K_nq z_aq + al_nq (q < Q), be_nq (q < Q)]  so that  D1[(n,a), b] + C_na = log2 v_nab  with the
// row constant C_na = sum_q (al z_aq + be z_aq^2) + B_n (returned; -inf for padded a / datapoints).
template <int Q>
__device__ __forceinline__ float build_a1_row(const TCLayout& L, const Rows& R, int lane, const float* za,
                                              bool valid_a, float* a1, int r) {
  constexpr int KV = (2 * Q + 7) / 8 * 8;
  float z[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) z[q] = za[q];
  float c = R.b2[lane];
#pragma unroll
  for (int j = 0; j < KV; j += 4) {
    float h[4], l[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = j + u;
      float x = 0.f;
      if (valid_a && k < 2 * Q) {
        if (k < Q) {
          const float al = R.al[k * 32 + lane];
          x = fmaf(R.kk[k * 32 + lane], z[k % Q], al);
          c = fmaf(al, z[k % Q], c);
        } else {
          const float be = R.be[(k - Q) * 32 + lane];
          x = be;
          c = fmaf(be * z[(k - Q) % Q], z[(k - Q) % Q], c);
        }
      }
      h[u] = tc::tf32_hi(x);
      l[u] = x - h[u];
    }
    if (j < L.k1) {
      *reinterpret_cast<float4*>(a1 + tc::canon(r, j, L.k1)) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(a1 + 128 * L.k1 + tc::canon(r, j, L.k1)) = make_float4(l[0], l[1], l[2], l[3]);
    }
  }
  return valid_a ? c : -CUDART_INF_F;
}

// Issue the 3xTF32 MMA1 of one tile: D1 = A1 B1^T (hi.hi + hi.lo + lo.hi).
template <int Q>
__device__ __forceinline__ void issue_mma1(const TCLayout& L, uint32_t d1, const float* a1, const float* b1) {
  constexpr int KS = (2 * Q + 7) / 8;  // K-steps of 8
  const uint32_t idesc = tc::idesc_tf32(128, L.n1);
  const uint64_t a_hi = tc::desc(tc::smem_u32(a1), L.k1), a_lo = tc::desc(tc::smem_u32(a1) + 128 * L.k1 * 4, L.k1);
  const uint64_t b_hi = tc::desc(tc::smem_u32(b1), L.k1), b_lo = tc::desc(tc::smem_u32(b1) + L.n1 * L.k1 * 4, L.k1);
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const uint64_t a = (t == 2) ? a_lo : a_hi, b = (t == 1) ? b_lo : b_hi;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) tc::mma_ss(d1, a + 16 * ks, b + 16 * ks, idesc, (t | ks) ? 1u : 0u);
  }
}

size_t fwd_tc_smem_bytes(const PsiConst& P) {
  const TCLayout L = tc_layout(P.q, P.m);
  size_t f = size_t(P.mv) * P.qv + rows_floats(P.qv) + 2 * size_t(L.n1) * L.k1 + kPipesF * 2 * 128 * size_t(L.k1);
  return f * 4 + 64 * sizeof(double) + 64;
}

// =============================================================================================
// Forward (statistics pass) on tensor cores.
// =============================================================================================
template <int Q>
__global__ void __launch_bounds__(kThreadsF, 1)
    psi_fwd_tc_kernel(PsiConst P, int64_t nchunks, double* __restrict__ part, int64_t pstride, int* err_flag) {
  extern __shared__ __align__(1024) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, nthr = blockDim.x;
  const int m = P.m, mv = P.mv, qv = P.qv, d = P.d, dv = P.dv;
  const TCLayout L = tc_layout(P.q, m);
  float* p = sm;
  float* B1 = p;  // 1024-aligned base keeps every operand tile 16-byte aligned
  p += 2 * L.n1 * L.k1;
  float* A1 = p;
  p += kPipesF * 2 * 128 * L.k1;
  float* Zc = p;
  p += mv * qv;
  Rows R = carve_rows(p, qv);
  double* red = reinterpret_cast<double*>(p);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(red + 64);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + kPipesF);

  for (int i = tid; i < mv * qv; i += nthr) Zc[i] = P.zc[i];
  __syncthreads();
  build_b1(P, L, Zc, B1);
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  if (tid == 0) {
    for (int i = 0; i < kPipesF; ++i) tc::mbar_init(&mbar[i], 1);
    tc::mbar_fence_init();
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  const int pipe = warp >> 2, wq = warp & 3;
  const uint32_t d1 = tmem + pipe * 128;
  const uint32_t lane_off = uint32_t(32 * wq) << 16;
  float* a1 = A1 + pipe * 2 * 128 * L.k1;
  uint32_t phase = 0;
  const int MT = (m + 3) >> 2;
  const int64_t npairs = int64_t(m) * (m + 1) / 2;
  double* const cta_part = part + int64_t(blockIdx.x) * pstride;
  double* const phi_part = cta_part + 2;
  (void)npairs;
  (void)d;
  (void)dv;

  double kl_acc = 0.0;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int64_t n0 = chunk * 32;
    TCP_MARK(tp0);
    load_rows<Q>(P, n0, R, P.expected ? &kl_acc : nullptr, err_flag);
    __syncthreads();
    TCP_ADD(0, tp0);

    // ---- psi2 on the tensor cores: this pipeline's row tiles ----
    {
      for (int t = pipe; t < MT; t += kPipesF) {
        const int a = 4 * t + wq;
        const bool va = a < m;
        TCP_MARK(tp1);
        const float La = build_a1_row<Q>(L, R, lane, Zc + (va ? a : 0) * qv, va, a1, 32 * wq + lane);
        tc::fence_async_smem();
        tc::fence_before();
        tc::named_sync(1 + pipe, 128);
        if (wq == 0 && lane == 0) {
          tc::fence_after();
          issue_mma1<Q>(L, d1, a1, B1);
          tc::commit(&mbar[pipe]);
        }
        TCP_ADD(1, tp1);
        TCP_MARK(tp2);
        tc::mbar_wait(&mbar[pipe], phase);
        phase ^= 1;
        tc::fence_after();
        TCP_ADD(2, tp2);
        TCP_MARK(tp3);
        const int c0 = (4 * t) & ~31;
        const int cfull = c0 + ((m - c0) & ~31);  // end of the full 32-column chunks
        uint32_t r[32];
        if (c0 < cfull) tc::ld32(d1 + lane_off + c0, r);
        for (int c = c0; c < cfull; c += 32) {
          tc::ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (c + 32 < cfull) tc::ld32(d1 + lane_off + c + 32, r);  // prefetch the next chunk
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int b = c + j;
            v[j] = (b >= a) ? ex2(v[j] + La) : 0.f;
          }
          const float tot = reduce_scatter<32>(v, lane);
          const int b = c + lane;
          if (va && b >= a) atomicAdd(phi_part + pair_index(a, b, m), double(tot));
        }
        for (int c = cfull; c < m; c += 8) {
          uint32_t r8[8];
          tc::ld8(d1 + lane_off + c, r8);
          tc::ld_wait();
          float v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int b = c + j;
            v[j] = (b >= a && b < m) ? ex2(__uint_as_float(r8[j]) + La) : 0.f;
          }
          const float tot = reduce_scatter<8>(v, lane);
          const int b = c + ((lane >> 2) & 7);
          if (va && b >= a && b < m && (lane & 3) == 0) atomicAdd(phi_part + pair_index(a, b, m), double(tot));
        }
        TCP_ADD(3, tp3);
        if (P.prof && wq == 0 && lane == 0) atomicAdd(P.prof + 8, 1ull);
      }
    }
    TCP_MARK(tp7);
    __syncthreads();
    TCP_ADD(7, tp7);
  }
  kl_acc = warp_sum_d(kl_acc);
  if (lane == 0) red[32 + warp] = kl_acc;
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
  if (tid == 0) {
    double s2 = 0.0;
    for (int i = 0; i < nw; ++i) s2 += red[32 + i];
    cta_part[1] = s2;  // yy and Psi come from psi1_fwd_kernel rows
  }
}

__global__ void fwd_reduce_tc(const double* __restrict__ part, int64_t pstride, int nparts, int64_t count,
                              double* __restrict__ packed, double phi_val, double n_count) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < count; k += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nparts; ++c) s += part[c * pstride + k];
    if (k == 0)
      packed[1] = s;
    else if (k == 1)
      packed[3] = s;
    else
      packed[k + 2] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    packed[0] = phi_val;
    packed[2] = n_count;
  }
}

// LaunchGeom.grid of the TC passes = partial rows (psi2 CTAs + psi1 rows), for buffer sizing.
template <int Q>
int plan_fwd_tc_q(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  const size_t smem = fwd_tc_smem_bytes(P);
  auto kern = psi_fwd_tc_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  const int64_t nchunks = (P.n + 31) / 32;
  const int g2 = int(std::min<int64_t>(nchunks, num_sms));
  *geom = LaunchGeom{g2 + psi1_fwd_rows(P, num_sms), kThreadsF, smem};
  return 0;
}

unsigned long long* tc_profile_buffer();
void tc_profile_report(const char* what, cudaStream_t st);

template <int Q>
int launch_fwd_tc_q(const PsiConst& P0, double* part, double* packed, int* err_flag, int num_sms, cudaStream_t st,
                    LaunchGeom* geom, cudaEvent_t e0, cudaEvent_t e1) {
  PsiConst P = P0;
  P.prof = tc_profile_buffer();
  LaunchGeom g{};
  if (int rc = plan_fwd_tc_q<Q>(P, num_sms, &g)) return rc;
  const int64_t nchunks = (P.n + 31) / 32;
  const int64_t pstride = fwd_part_count(P.m, P.d);
  const int g2 = int(std::min<int64_t>(nchunks, num_sms)), g1 = g.grid - g2;
  if (nchunks > 0) {
    if (cudaMemsetAsync(part, 0, sizeof(double) * pstride * g.grid, st) != cudaSuccess) return 3;
    if (e0) cudaEventRecord(e0, st);
    psi_fwd_tc_kernel<Q><<<g2, g.threads, g.smem, st>>>(P, nchunks, part, pstride, err_flag);
    g_tc_launches.fetch_add(1);
    if (int rc = psi1_forward(P, part + int64_t(g2) * pstride, pstride, g1, err_flag, st, 0)) return rc;
    if (e1) cudaEventRecord(e1, st);
  }
  fwd_reduce_tc<<<int((pstride + 255) / 256), 256, 0, st>>>(part, pstride, nchunks > 0 ? g.grid : 0, pstride,
                                                            packed, double(P.n) * P.variance_d, double(P.n));
  g_tc_launches.fetch_add(1);
  tc_profile_report("fwd", st);
  if (geom) *geom = g;
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}


// =============================================================================================
// Backward (gradient pass): MMA1 on the tensor cores for the exponent cross term, SIMT for
// G = U_ab ex2(s) and the accumulations R_na = sum_b G, S_naq = sum_b G z_bq.
// A tile is 32 datapoints x 8 inducing points: warp quadrant wq owns rows (n, a = 8t + wq) in
// TMEM columns [0, 128) and (n, a + 4) in [128, 256), so one broadcast load of z_b feeds a
// packed fma.rn.f32x2 over the two rows.  TMEM: 256 columns per pipeline, 2 pipelines.
// =============================================================================================
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}

size_t bwd_tc_smem_bytes(const PsiConst& P, int Q) {
  const TCLayout L = tc_layout(P.q, P.m);
  size_t f = 2 * size_t(L.n1) * L.k1 + kPipes * 2 * (2 * 128 * size_t(L.k1)) + size_t(P.mv) * P.qv +
             rows_floats(P.qv) + size_t(P.mv) * P.mv;
  // the per-warp merge buffer aliases the A1 operand buffers (used only after the tile loop)
  const size_t a1f = kPipes * 2 * (2 * 128 * size_t(L.k1)), accf = size_t(kThreadsTC / 32) * (1 + 3 * Q) * 32;
  if (accf > a1f) f += accf - a1f;
  return f * 4 + (Q + 1) * 32 * sizeof(double) + 64;
}

template <int Q>
__global__ void __launch_bounds__(kThreadsTC, 1)
    psi_bwd_tc_kernel(PsiConst P, BwdConst B, int64_t nchunks, double* __restrict__ part, int64_t pstride) {
  constexpr int NACC = 1 + 3 * Q;
  constexpr int T0 = 0, Y1 = 1, Y2 = 1 + Q, XX = 1 + 2 * Q;
  constexpr int Q4 = (Q + 3) / 4;
  extern __shared__ __align__(1024) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, nthr = blockDim.x;
  const int m = P.m, mv = P.mv, qv = P.qv;
  const TCLayout L = tc_layout(P.q, m);
  float* p = sm;
  float* B1 = p;
  p += 2 * L.n1 * L.k1;
  float* A1 = p;  // [pipe][group][hi/lo][128 x k1]
  p += kPipes * 2 * (2 * 128 * L.k1);
  float* Zc = p;
  p += mv * qv;
  Rows R = carve_rows(p, qv);
  float* Us = p;  // U = dL/dPhi, [mv][mv] (symmetric, zero padded)
  p += mv * mv;
  float* acc = A1;  // per-warp per-datapoint merge buffer, aliases A1 (only used after the tile loop)
  {
    const int a1f = kPipes * 2 * (2 * 128 * L.k1), accf = nw * NACC * 32;
    if (accf > a1f) p += accf - a1f;
  }
  double* dacc = reinterpret_cast<double*>(p);  // [(Q+1)][32]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(dacc + (Q + 1) * 32);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + kPipes);

  for (int i = tid; i < mv * qv; i += nthr) Zc[i] = P.zc[i];
  for (int i = tid; i < mv * mv; i += nthr) Us[i] = B.u[i];
  for (int i = tid; i < (Q + 1) * 32; i += nthr) dacc[i] = 0.0;
  __syncthreads();
  build_b1(P, L, Zc, B1);
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  if (tid == 0) {
    for (int i = 0; i < kPipes; ++i) tc::mbar_init(&mbar[i], 1);
    tc::mbar_fence_init();
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  const int pipe = warp >> 2, wq = warp & 3;
  const uint32_t base = tmem + pipe * 256;
  const uint32_t lane_off = uint32_t(32 * wq) << 16;
  float* a1g0 = A1 + pipe * 2 * (2 * 128 * L.k1);
  float* a1g1 = a1g0 + 2 * 128 * L.k1;
  uint32_t ph = 0;
  const int MT8 = (m + 7) >> 3;  // tiles of 8 inducing points
  double* const cta_part = part + int64_t(blockIdx.x) * pstride;
  double* const dz_part = cta_part + 1 + P.q;
  const double inv_var = 1.0 / P.variance_d;

  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int64_t n0 = chunk * 32, n = n0 + lane;
    const bool valid = n < P.n;
    TCP_MARK(tp0);
    load_rows<Q>(P, n0, R, nullptr, nullptr);
    __syncthreads();
    TCP_ADD(0, tp0);

    float t0 = 0.f, y1[Q], y2[Q], xq[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) y1[q] = y2[q] = xq[q] = 0.f;
    for (int t = pipe; t < MT8; t += kPipes) {
      const int a0 = 8 * t + wq, a1i = a0 + 4;
      const bool va0 = a0 < m, va1 = a1i < m;
      const int ac0 = va0 ? a0 : 0, ac1 = va1 ? a1i : 0;
      TCP_MARK(tp1);
      // row constants C_na (padded rows a >= M get -inf so their G, R, S vanish)
      const float2 La = make_float2(build_a1_row<Q>(L, R, lane, Zc + ac0 * qv, va0, a1g0, 32 * wq + lane),
                                    build_a1_row<Q>(L, R, lane, Zc + ac1 * qv, va1, a1g1, 32 * wq + lane));
      tc::fence_async_smem();
      tc::fence_before();
      tc::named_sync(1 + pipe, 128);
      if (wq == 0 && lane == 0) {
        tc::fence_after();
        issue_mma1<Q>(L, base, a1g0, B1);
        issue_mma1<Q>(L, base + 128, a1g1, B1);
        tc::commit(&mbar[pipe]);
      }
      TCP_ADD(1, tp1);
      TCP_MARK(tp2);
      tc::mbar_wait(&mbar[pipe], ph);
      ph ^= 1;
      tc::fence_after();
      TCP_ADD(2, tp2);
      TCP_MARK(tp3);
      const float* u0 = Us + ac0 * mv;  // U symmetric: rows a0, a0+4
      const float* u1 = Us + ac1 * mv;
      float2 Racc = make_float2(0.f, 0.f), Sacc[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) Sacc[q] = make_float2(0.f, 0.f);
      // one column b for the two rows of this thread
      auto column = [&](int b, float d0, float d1, float ua, float ub) {
        const float g0 = ua * ex2(d0 + La.x), g1 = ub * ex2(d1 + La.y);
        Racc.x += g0;
        Racc.y += g1;
        float z[Q];
        load_z<Q>(Zc + b * qv, z);
        const float2 g = make_float2(g0, g1);
#pragma unroll
        for (int q = 0; q < Q; ++q) Sacc[q] = fma2(g, make_float2(z[q], z[q]), Sacc[q]);
      };
      // full 16-column chunks: no bound checks
      const int cfull = m & ~15;
      for (int c = 0; c < cfull; c += 16) {
        uint32_t r0[16], r1[16];
        tc::ld16(base + lane_off + c, r0);
        tc::ld16(base + 128 + lane_off + c, r1);
        tc::ld_wait();
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const float4 ua = *reinterpret_cast<const float4*>(u0 + c + j);
          const float4 ub = *reinterpret_cast<const float4*>(u1 + c + j);
          column(c + j + 0, __uint_as_float(r0[j + 0]), __uint_as_float(r1[j + 0]), ua.x, ub.x);
          column(c + j + 1, __uint_as_float(r0[j + 1]), __uint_as_float(r1[j + 1]), ua.y, ub.y);
          column(c + j + 2, __uint_as_float(r0[j + 2]), __uint_as_float(r1[j + 2]), ua.z, ub.z);
          column(c + j + 3, __uint_as_float(r0[j + 3]), __uint_as_float(r1[j + 3]), ua.w, ub.w);
        }
      }
      if (cfull < m) {  // tail (< 16 columns; U and Zc are padded to mv, so b < mv reads stay in range)
        uint32_t r0[16], r1[16];
        tc::ld16(base + lane_off + cfull, r0);
        tc::ld16(base + 128 + lane_off + cfull, r1);
        tc::ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int b = cfull + j;
          if (b < m) column(b, __uint_as_float(r0[j]), __uint_as_float(r1[j]), u0[b], u1[b]);
        }
      }
      TCP_ADD(3, tp3);
      TCP_MARK(tp6);
      // contractions for the two rows (natural-log units; G carries U and v)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = h ? a1i : a0;
        const bool va = h ? va1 : va0;
        const int ac = h ? ac1 : ac0;
        const float Ra = h ? Racc.y : Racc.x;
        t0 += Ra;
        float vals[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const float Sa = h ? Sacc[q].y : Sacc[q].x;
          const float z = Zc[ac * qv + q];
          y1[q] = fmaf(z, Ra, y1[q]);
          y2[q] = fmaf(z * z, Ra, y2[q]);
          xq[q] = fmaf(z, Sa, xq[q]);
          const float mu = R.mu[q * 32 + lane], d2 = R.d2[q * 32 + lane];
          const float kn = R.sv[q * 32 + lane] * P.il2[q] * d2;
          const float c2 = 0.5f * (P.il2[q] + d2);
          vals[q] = 2.f * (fmaf(d2, mu, -c2 * z) * Ra + kn * Sa);
        }
        constexpr int QR = Q <= 8 ? 8 : (Q <= 16 ? 16 : 32);
        float vr[QR];
#pragma unroll
        for (int i = 0; i < QR; ++i) vr[i] = (i < Q) ? vals[i % Q] : 0.f;
        const float tot = reduce_scatter<QR>(vr, lane);
        const int shift = QR == 8 ? 2 : (QR == 16 ? 1 : 0);
        const int qi = lane >> shift;
        if (va && qi < P.q && (lane & ((1 << shift) - 1)) == 0)
          atomicAdd(dz_part + a + int64_t(qi) * m, double(tot));
      }
      TCP_ADD(6, tp6);
      if (P.prof && wq == 0 && lane == 0) atomicAdd(P.prof + 8, 1ull);
    }
    (void)Q4;
    TCP_MARK(tp7);
    __syncthreads();  // every pipeline is done with its A1 buffers (acc aliases them)
    {
      float* accw = acc + warp * NACC * 32;
      accw[T0 * 32 + lane] = t0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        accw[(Y1 + q) * 32 + lane] = y1[q];
        accw[(Y2 + q) * 32 + lane] = y2[q];
        accw[(XX + q) * 32 + lane] = xq[q];
      }
    }
    __syncthreads();
    for (int q = warp; q < P.q; q += nw) {
      if (!valid) continue;
      double T = 0, A1s = 0, A2s = 0, X = 0;
      for (int w2 = 0; w2 < nw; ++w2) {
        const float* aw = acc + w2 * NACC * 32;
        T += aw[T0 * 32 + lane];
        A1s += aw[(Y1 + q) * 32 + lane];
        A2s += aw[(Y2 + q) * 32 + lane];
        X += aw[(XX + q) * 32 + lane];
      }
      const double mu = R.mu[q * 32 + lane], sv = R.sv[q * 32 + lane];
      const double l = P.ls[q], l2 = l * l, il2 = 1.0 / l2, il3 = il2 / l;
      const double d2 = 1.0 / (2.0 * sv + l2);
      const double dl = T * (2.0 * sv * d2 / l + 2.0 * l * d2 * d2 * mu * mu) - 4.0 * l * d2 * d2 * mu * A1s +
                        A2s * (il3 + l * d2 * d2) - X * (il3 - l * d2 * d2);
      dacc[q * 32 + lane] += dl;
      if (q == 0) dacc[Q * 32 + lane] += 2.0 * T * inv_var;
      if (B.write_local) {  // psi1_bwd_kernel wrote the psi1 and KL parts first
        B.d_mu[q * B.ld_g + n] += -2.0 * d2 * mu * T + 2.0 * d2 * A1s;
        B.d_s[q * B.ld_g + n] += T * (-d2 + 2.0 * d2 * d2 * mu * mu) - 4.0 * d2 * d2 * mu * A1s + d2 * d2 * (A2s + X);
      }
    }
    __syncthreads();
    TCP_ADD(7, tp7);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
  if (tid <= Q) {
    double s = 0.0;
    for (int l2i = 0; l2i < 32; ++l2i) s += dacc[tid * 32 + l2i];
    if (tid < P.q)
      cta_part[1 + tid] = s;
    else if (tid == Q)
      cta_part[0] = s;
  }
}

__global__ void bwd_reduce_tc(const double* __restrict__ part, int64_t pstride, int nparts, int64_t count,
                              double* __restrict__ packed, double dvar0) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < count; k += int64_t(gridDim.x) * blockDim.x) {
    double s = (k == 0) ? dvar0 : 0.0;
    for (int c = 0; c < nparts; ++c) s += part[c * pstride + k];
    packed[k] = s;
  }
}

template <int Q>
int plan_bwd_tc_q(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  const size_t smem = bwd_tc_smem_bytes(P, Q);
  if (smem > 227 * 1024) return 1;
  auto kern = psi_bwd_tc_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  const int64_t nchunks = (P.n + 31) / 32;
  const int g2 = int(std::min<int64_t>(nchunks, num_sms));
  *geom = LaunchGeom{g2 + psi1_bwd_rows(P, num_sms), kThreadsTC, smem};
  return 0;
}

unsigned long long* tc_profile_buffer() {
  static unsigned long long* buf = nullptr;
  static const bool on = getenv("SGPX_TC_PROFILE") != nullptr;
  if (on && !buf) {
    cudaMalloc(&buf, 16 * sizeof(unsigned long long));
    cudaMemset(buf, 0, 16 * sizeof(unsigned long long));
  }
  return on ? buf : nullptr;
}

void tc_profile_report(const char* what, cudaStream_t st) {
  unsigned long long* buf = tc_profile_buffer();
  if (!buf) return;
  unsigned long long h[16];
  cudaStreamSynchronize(st);
  cudaMemcpy(h, buf, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"prologue", "a1+bar", "mma1_wait", "elements", "mma2_issue", "mma2_wait", "contract",
                         "epilogue"};
  fprintf(stderr, "[tc-profile %s] tiles/pipe-sum=%llu:", what, h[8]);
  unsigned long long tot = 0;
  for (int i = 0; i < 8; ++i) tot += h[i];
  for (int i = 0; i < 8; ++i) fprintf(stderr, " %s=%.1f%%", names[i], 100.0 * h[i] / (tot ? tot : 1));
  fprintf(stderr, " (cycles/tile %.0f)\n", double(tot) / double(h[8] ? h[8] : 1));
  cudaMemset(buf, 0, sizeof(h));
}

template <int Q>
int launch_bwd_tc_q(const PsiConst& P0, const BwdConst& B, double* part, double* packed, int num_sms, cudaStream_t st,
                    LaunchGeom* geom, cudaEvent_t e0, cudaEvent_t e1) {
  PsiConst P = P0;
  P.prof = tc_profile_buffer();
  LaunchGeom g{};
  if (int rc = plan_bwd_tc_q<Q>(P, num_sms, &g)) return rc;
  const int64_t nchunks = (P.n + 31) / 32;
  const int64_t pstride = bwd_part_count(P.m, P.q);
  const int g2 = int(std::min<int64_t>(nchunks, num_sms)), r1 = g.grid - g2;
  if (nchunks > 0) {
    if (cudaMemsetAsync(part, 0, sizeof(double) * pstride * g.grid, st) != cudaSuccess) return 3;
    if (e0) cudaEventRecord(e0, st);
    // psi1 first: it writes d_mu / d_s (psi1 + KL parts); the psi2 kernel accumulates into them
    if (int rc = psi1_backward(P, B, part + int64_t(g2) * pstride, pstride, r1, st)) return rc;
    psi_bwd_tc_kernel<Q><<<g2, g.threads, g.smem, st>>>(P, B, nchunks, part, pstride);
    g_tc_launches.fetch_add(1);
    if (e1) cudaEventRecord(e1, st);
  }
  bwd_reduce_tc<<<int((pstride + 255) / 256), 256, 0, st>>>(part, pstride, nchunks > 0 ? g.grid : 0, pstride,
                                                            packed, B.d_phi * double(P.n));
  g_tc_launches.fetch_add(1);
  tc_profile_report("bwd", st);
  if (geom) *geom = g;
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

bool tc_supported(const PsiConst& P) { return P.m >= 1 && P.m <= 128 && P.q >= 1 && P.q <= 32; }

// Two-level fixed-order reduction of `rows` partial rows: row groups in parallel (level 1), then
// the group sums in ascending order (level 2).  tmp: kReduceGroups * pstride doubles.
namespace {
constexpr int kReduceGroups = 64;
__global__ void rows_partial_kernel(const double* __restrict__ part, int64_t pstride, int rows, int groups,
                                    double* __restrict__ tmp) {
  const int g = blockIdx.y;
  const int r0 = int(int64_t(g) * rows / groups), r1 = int(int64_t(g + 1) * rows / groups);
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < pstride; k += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int r = r0; r < r1; ++r) s += part[int64_t(r) * pstride + k];
    tmp[int64_t(g) * pstride + k] = s;
  }
}
__global__ void rows_final_bwd_kernel(const double* __restrict__ tmp, int groups, int64_t pstride,
                                      double* __restrict__ packed, double dvar0) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < pstride; k += int64_t(gridDim.x) * blockDim.x) {
    double s = k == 0 ? dvar0 : 0.0;
    for (int g = 0; g < groups; ++g) s += tmp[int64_t(g) * pstride + k];
    packed[k] = s;
  }
}
}  // namespace

int64_t bwd_reduce_tmp_doubles(int64_t pstride) { return int64_t(kReduceGroups) * pstride; }

int bwd_reduce_rows(const double* part, int64_t pstride, int rows, double* packed, double dvar0, double* tmp,
                    void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int groups = std::max(1, std::min(kReduceGroups, rows));
  const int cb = int(std::min<int64_t>((pstride + 255) / 256, 64));
  rows_partial_kernel<<<dim3(cb, groups), 256, 0, st>>>(part, pstride, rows, groups, tmp);
  rows_final_bwd_kernel<<<cb, 256, 0, st>>>(tmp, groups, pstride, packed, dvar0);
  g_tc_launches.fetch_add(2);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Backward TMEM budget per pipeline: 2 n1 + n2 <= 256 columns.
bool tc_backward_fits(const PsiConst& P) {
  return tc_supported(P) && P.q <= 16 && bwd_tc_smem_bytes(P, instantiated_q(P.q)) <= 227 * 1024;
}
bool tc_backward_available() { return true; }

#define SGPX_TC_DISPATCH(FN, ...)                      \
  switch (instantiated_q(P.q)) {                       \
    case 1: return FN<1>(__VA_ARGS__);                 \
    case 2: return FN<2>(__VA_ARGS__);                 \
    case 3: return FN<3>(__VA_ARGS__);                 \
    case 4: return FN<4>(__VA_ARGS__);                 \
    case 5: return FN<5>(__VA_ARGS__);                 \
    case 6: return FN<6>(__VA_ARGS__);                 \
    case 8: return FN<8>(__VA_ARGS__);                 \
    case 10: return FN<10>(__VA_ARGS__);               \
    case 12: return FN<12>(__VA_ARGS__);               \
    case 16: return FN<16>(__VA_ARGS__);               \
    default: return 1;                                 \
  }

int plan_backward_tc(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  SGPX_TC_DISPATCH(plan_bwd_tc_q, P, num_sms, geom)
}

int psi_backward_tc(const PsiConst& P, const BwdConst& B, double* part, double* packed, int num_sms, void* stream,
                    LaunchGeom* geom, void* ev_begin, void* ev_end) {
  SGPX_TC_DISPATCH(launch_bwd_tc_q, P, B, part, packed, num_sms, static_cast<cudaStream_t>(stream), geom,
                   cudaEvent_t(ev_begin), cudaEvent_t(ev_end))
}


int plan_forward_tc(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  switch (instantiated_q(P.q)) {
    case 1: return plan_fwd_tc_q<1>(P, num_sms, geom);
    case 2: return plan_fwd_tc_q<2>(P, num_sms, geom);
    case 3: return plan_fwd_tc_q<3>(P, num_sms, geom);
    case 4: return plan_fwd_tc_q<4>(P, num_sms, geom);
    case 5: return plan_fwd_tc_q<5>(P, num_sms, geom);
    case 6: return plan_fwd_tc_q<6>(P, num_sms, geom);
    case 8: return plan_fwd_tc_q<8>(P, num_sms, geom);
    case 10: return plan_fwd_tc_q<10>(P, num_sms, geom);
    case 12: return plan_fwd_tc_q<12>(P, num_sms, geom);
    case 16: return plan_fwd_tc_q<16>(P, num_sms, geom);
    case 20: return plan_fwd_tc_q<20>(P, num_sms, geom);
    case 24: return plan_fwd_tc_q<24>(P, num_sms, geom);
    case 32: return plan_fwd_tc_q<32>(P, num_sms, geom);
    default: return 1;
  }
}

int psi_forward_tc(const PsiConst& P, double* part, double* packed, int* err_flag, int num_sms, void* stream,
                   LaunchGeom* geom, void* ev_begin, void* ev_end) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t e0 = cudaEvent_t(ev_begin), e1 = cudaEvent_t(ev_end);
  switch (instantiated_q(P.q)) {
    case 1: return launch_fwd_tc_q<1>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 2: return launch_fwd_tc_q<2>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 3: return launch_fwd_tc_q<3>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 4: return launch_fwd_tc_q<4>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 5: return launch_fwd_tc_q<5>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 6: return launch_fwd_tc_q<6>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 8: return launch_fwd_tc_q<8>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 10: return launch_fwd_tc_q<10>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 12: return launch_fwd_tc_q<12>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 16: return launch_fwd_tc_q<16>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 20: return launch_fwd_tc_q<20>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 24: return launch_fwd_tc_q<24>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    case 32: return launch_fwd_tc_q<32>(P, part, packed, err_flag, num_sms, st, geom, e0, e1);
    default: return 1;
  }
}

}  // namespace sgpx
