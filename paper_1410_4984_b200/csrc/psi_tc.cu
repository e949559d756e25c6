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

#include "psi_common.cuh"
#include "psi_kernels.cuh"
#include "tc_util.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;
std::atomic<int64_t> g_tc_launches{0};

namespace {
using namespace dev;

constexpr int kPipes = 2;
constexpr int kThreadsTC = 128 * kPipes;

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Sum of v[i] over the warp for K values per lane (K in {8, 16, 32}): lane ends up holding
// the total of index lane >> (5 - log2 K).
template <int K>
__device__ __forceinline__ float reduce_scatter(float (&v)[K], int lane) {
  int n = K;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (n > 1) {
      const int h = n >> 1;
      const bool hi = lane & off;
#pragma unroll
      for (int i = 0; i < K / 2; ++i) {
        if (i < h) {
          const float send = hi ? v[i] : v[i + h];
          const float keep = hi ? v[i + h] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      n = h;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  return v[0];
}

struct TCLayout {
  int k1;    // MMA1 K (Q rounded to 8)
  int n1;    // MMA1 N (M rounded to 16), <= 128
  int k2;    // MMA2 K (M rounded to 8)
  int n2;    // MMA2 N (Q+1 rounded to 16)
};

__host__ __device__ inline TCLayout tc_layout(int q, int m) {
  return TCLayout{round_up(q, 8), round_up(m, 16), round_up(m, 8), round_up(q + 1, 16)};
}

// B1 = centred Z as the K-major B operand (N1 rows b, K1 columns q), hi and lo planes.
__device__ __forceinline__ void build_b1(const PsiConst& P, const TCLayout& L, const float* Zc, float* b1) {
  const int tot = L.n1 * L.k1;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    const int b = i / L.k1, q = i - b * L.k1;
    const float z = (b < P.m && q < P.q) ? Zc[b * P.qv + q] : 0.f;
    const float h = tc::tf32_hi(z);
    b1[tc::canon(b, q, L.k1)] = h;
    b1[L.n1 * L.k1 + tc::canon(b, q, L.k1)] = z - h;
  }
}

// A1 rows of one tile: row r = 32*wq + lane <-> (datapoint lane, inducing a), value K_nq z_aq.
template <int Q>
__device__ __forceinline__ void build_a1_row(const TCLayout& L, const float (&kk)[Q], const float* za, bool valid_a,
                                             float* a1, int r) {
  constexpr int QV = (Q + 7) / 8 * 8;
#pragma unroll
  for (int j = 0; j < QV; j += 4) {
    float h[4], l[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = j + u;
      const float x = (q < Q && valid_a) ? kk[q % Q] * za[q % Q] : 0.f;
      h[u] = tc::tf32_hi(x);
      l[u] = x - h[u];
    }
    if (j < L.k1) {
      *reinterpret_cast<float4*>(a1 + tc::canon(r, j, L.k1)) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(a1 + 128 * L.k1 + tc::canon(r, j, L.k1)) = make_float4(l[0], l[1], l[2], l[3]);
    }
  }
}

// Issue the 3xTF32 MMA1 of one tile: D1 = A1 B1^T (hi.hi + hi.lo + lo.hi).
__device__ __forceinline__ void issue_mma1(const TCLayout& L, uint32_t d1, const float* a1, const float* b1) {
  const uint32_t idesc = tc::idesc_tf32(128, L.n1);
  const uint32_t a_hi = tc::smem_u32(a1), a_lo = a_hi + 128 * L.k1 * 4;
  const uint32_t b_hi = tc::smem_u32(b1), b_lo = b_hi + L.n1 * L.k1 * 4;
  uint32_t acc = 0;
  for (int t = 0; t < 3; ++t) {
    const uint32_t a = (t == 2) ? a_lo : a_hi, b = (t == 1) ? b_lo : b_hi;
    for (int ks = 0; ks < L.k1 / 8; ++ks) {
      tc::mma_ss(d1, tc::desc(a + ks * 256, L.k1), tc::desc(b + ks * 256, L.k1), idesc, acc);
      acc = 1;
    }
  }
}

size_t fwd_tc_smem_bytes(const PsiConst& P) {
  const TCLayout L = tc_layout(P.q, P.m);
  size_t f = size_t(P.mv) * P.qv + rows_floats(P.qv) + size_t(P.mv) * 32 * 2 + 32 * size_t(P.dv) +
             2 * size_t(L.n1) * L.k1 + kPipes * 2 * 128 * size_t(L.k1);
  return f * 4 + 64 * sizeof(double) + 64;
}

// =============================================================================================
// Forward (statistics pass) on tensor cores.
// =============================================================================================
template <int Q>
__global__ void __launch_bounds__(kThreadsTC, 1)
    psi_fwd_tc_kernel(PsiConst P, int64_t nchunks, double* __restrict__ part, int64_t pstride, int* err_flag) {
  extern __shared__ __align__(1024) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, nthr = blockDim.x;
  const int m = P.m, mv = P.mv, qv = P.qv, d = P.d, dv = P.dv;
  const TCLayout L = tc_layout(P.q, m);
  float* p = sm;
  float* B1 = p;  // 1024-aligned base keeps every operand tile 16-byte aligned
  p += 2 * L.n1 * L.k1;
  float* A1 = p;
  p += kPipes * 2 * 128 * L.k1;
  float* Zc = p;
  p += mv * qv;
  Rows R = carve_rows(p, qv);
  float* Ls = p;
  p += mv * 32;
  float* V1s = p;
  p += 32 * mv;
  float* Ys = p;
  p += 32 * dv;
  double* red = reinterpret_cast<double*>(p);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(red + 64);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + kPipes);

  for (int i = tid; i < mv * qv; i += nthr) Zc[i] = P.zc[i];
  __syncthreads();
  build_b1(P, L, Zc, B1);
  if (warp == 0) tc::tmem_alloc(tmem_slot, 256);
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
  const uint32_t d1 = tmem + pipe * 128;
  const uint32_t lane_off = uint32_t(32 * wq) << 16;
  float* a1 = A1 + pipe * 2 * 128 * L.k1;
  uint32_t phase = 0;
  const int MT = (m + 3) >> 2;
  const int64_t npairs = int64_t(m) * (m + 1) / 2;
  double* const cta_part = part + int64_t(blockIdx.x) * pstride;
  double* const phi_part = cta_part + 2;
  double* const psi_part = phi_part + npairs;
  const int DT = dv >> 2;
  const int ntiles1 = (mv >> 2) * DT;

  double yy_acc = 0.0, kl_acc = 0.0;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int64_t n0 = chunk * 32, n = n0 + lane;
    const bool valid = n < P.n;
    load_rows<Q>(P, n0, R, P.expected ? &kl_acc : nullptr, err_flag);
    build_L<Q>(P, R, Zc, Ls);
    {  // psi1 values [n][m]
      float mu[Q], d1v[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        mu[q] = R.mu[q * 32 + lane];
        d1v[q] = R.d1[q * 32 + lane];
      }
      const float b1 = R.b1[lane];
      for (int mm = warp; mm < mv; mm += nw) {
        float v = 0.f;
        if (mm < m) {
          float z[Q];
          load_z<Q>(Zc + mm * qv, z);
          float e = 0.f;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const float df = mu[q] - z[q];
            e = fmaf(df * df, d1v[q], e);
          }
          v = ex2(fmaf(-0.5f * kLog2e, e, b1));
        }
        V1s[lane * mv + mm] = v;
      }
    }
    for (int dd = warp; dd < dv; dd += nw) {
      float yv = 0.f;
      if (dd < d && valid) {
        const double yd = P.y[dd * P.ld_y + n];
        if (!isfinite(yd)) atomicOr(err_flag, 1);
        yy_acc += yd * yd;
        yv = float(yd);
      }
      Ys[lane * dv + dd] = yv;
    }
    __syncthreads();

    // ---- psi2 on the tensor cores: this pipeline's row tiles ----
    {
      float kk[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) kk[q] = R.kk[q * 32 + lane];
      for (int t = pipe; t < MT; t += kPipes) {
        const int a = 4 * t + wq;
        const bool va = a < m;
        build_a1_row<Q>(L, kk, Zc + (va ? a : 0) * qv, va, a1, 32 * wq + lane);
        tc::fence_async_smem();
        tc::fence_before();
        tc::named_sync(1 + pipe, 128);
        if (wq == 0 && lane == 0) {
          tc::fence_after();
          issue_mma1(L, d1, a1, B1);
          tc::commit(&mbar[pipe]);
        }
        tc::mbar_wait(&mbar[pipe], phase);
        phase ^= 1;
        tc::fence_after();
        const float La = Ls[(va ? a : 0) * 32 + lane];
        const int c0 = (4 * t) & ~31;
        int c = c0;
        for (; c + 32 <= m; c += 32) {
          uint32_t r[32];
          tc::ld32(d1 + lane_off + c, r);
          tc::ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int b = c + j;
            const float s = __uint_as_float(r[j]) + La + Ls[b * 32 + lane];
            v[j] = (b >= a) ? ex2(s) : 0.f;
          }
          const float tot = reduce_scatter<32>(v, lane);
          const int b = c + lane;
          if (va && b >= a) atomicAdd(phi_part + pair_index(a, b, m), double(tot));
        }
        for (; c < m; c += 8) {
          uint32_t r[8];
          tc::ld8(d1 + lane_off + c, r);
          tc::ld_wait();
          float v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int b = c + j;
            const float s = __uint_as_float(r[j]) + La + Ls[min(b, mv - 1) * 32 + lane];
            v[j] = (b >= a && b < m) ? ex2(s) : 0.f;
          }
          const float tot = reduce_scatter<8>(v, lane);
          const int b = c + ((lane >> 2) & 7);
          if (va && b >= a && b < m && (lane & 3) == 0) atomicAdd(phi_part + pair_index(a, b, m), double(tot));
        }
      }
    }
    // ---- psi1: Psi = Psi1^T Y, 4 m x 4 d register tiles over the chunk ----
    for (int t = tid; t < ntiles1; t += nthr) {
      const int mt = t / DT, dt = t - mt * DT;
      float acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const float4 vv = *reinterpret_cast<const float4*>(V1s + k * mv + 4 * mt);
        const float4 yv = *reinterpret_cast<const float4*>(Ys + k * dv + 4 * dt);
        const float va4[4] = {vv.x, vv.y, vv.z, vv.w}, ya[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(va4[i], ya[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int mm = 4 * mt + i, dd = 4 * dt + j;
          if (mm < m && dd < d) atomicAdd(psi_part + mm + int64_t(dd) * m, double(acc[i][j]));
        }
    }
    __syncthreads();
  }
  yy_acc = warp_sum_d(yy_acc);
  kl_acc = warp_sum_d(kl_acc);
  if (lane == 0) {
    red[warp] = yy_acc;
    red[32 + warp] = kl_acc;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 256);
  }
  if (tid == 0) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < nw; ++i) {
      s1 += red[i];
      s2 += red[32 + i];
    }
    cta_part[0] = s1;
    cta_part[1] = s2;
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

template <int Q>
int plan_fwd_tc_q(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  const size_t smem = fwd_tc_smem_bytes(P);
  auto kern = psi_fwd_tc_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  const int64_t nchunks = (P.n + 31) / 32;
  *geom = LaunchGeom{int(std::min<int64_t>(nchunks, num_sms)), kThreadsTC, smem};
  return 0;
}

template <int Q>
int launch_fwd_tc_q(const PsiConst& P, double* part, double* packed, int* err_flag, int num_sms, cudaStream_t st,
                    LaunchGeom* geom, cudaEvent_t e0, cudaEvent_t e1) {
  LaunchGeom g{};
  if (int rc = plan_fwd_tc_q<Q>(P, num_sms, &g)) return rc;
  const int64_t nchunks = (P.n + 31) / 32;
  const int64_t pstride = fwd_part_count(P.m, P.d);
  if (g.grid > 0) {
    if (cudaMemsetAsync(part, 0, sizeof(double) * pstride * g.grid, st) != cudaSuccess) return 3;
    if (e0) cudaEventRecord(e0, st);
    psi_fwd_tc_kernel<Q><<<g.grid, g.threads, g.smem, st>>>(P, nchunks, part, pstride, err_flag);
    if (e1) cudaEventRecord(e1, st);
    g_tc_launches.fetch_add(1);
  }
  fwd_reduce_tc<<<int((pstride + 255) / 256), 256, 0, st>>>(part, pstride, g.grid, pstride, packed,
                                                            double(P.n) * P.variance_d, double(P.n));
  g_tc_launches.fetch_add(1);
  if (geom) *geom = g;
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

bool tc_supported(const PsiConst& P) { return P.m >= 1 && P.m <= 128 && P.q >= 1 && P.q <= 32; }
bool tc_backward_available() { return false; }
int plan_backward_tc(const PsiConst&, int, LaunchGeom*) { return 1; }
int psi_backward_tc(const PsiConst&, const BwdConst&, double*, double*, int, void*, LaunchGeom*, void*, void*) {
  return 1;
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
