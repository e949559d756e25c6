// psi_kernels.cu -- sm_100a psi-statistics forward / backward kernels.
//
// Reference hot path: proj/include/sgp/psi_stats.hpp:108-326 (detail::sweep_stats),
// plus the KL partial / KL gradients of Worker::pass (parallel.hpp:148-149, 163-166).
//
// Execution model:
//   * persistent CTAs; a CTA processes chunks of 32 datapoints, one datapoint
//     per lane; all warps of the CTA share the chunk's per-datapoint tables in
//     shared memory (Z, L_na, psi1 values, y tile),
//   * forward: warps split the upper triangle of 4x4 inducing-pair tiles; each
//     tile's 16 values are reduced over the 32 lanes (datapoints) with a
//     shuffle reduce-scatter and accumulated in fp64 (RED.ADD.F64) into a
//     CTA-private partial row; Psi = Psi1^T Y is a 4x4 register-tiled product
//     over the chunk,
//   * backward: warps own 4-row tiles of inducing indices a and sweep all b,
//     keeping the per-(n,a) sums R = sum_b G, S_q = sum_b G z_bq in registers;
//     per-datapoint contractions go to warp-private shared memory, per-a
//     contractions (dZ) are reduce-scattered over lanes into fp64 partials,
//   * every cross-CTA sum is fp64 and happens in fixed CTA order in a second
//     tiny kernel, so results are bitwise reproducible run to run.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "psi_common.cuh"
#include "psi_kernels.cuh"

namespace sgpx {
namespace {

std::atomic<int64_t> g_launches{0};
using namespace dev;

// =============================================================================
// Forward: phi-stats partials (yy, KL, Phi pairs, Psi) per CTA.
// =============================================================================
template <int Q>
__global__ void __launch_bounds__(256, 2)
    psi_fwd_kernel(PsiConst P, int64_t nchunks, double* __restrict__ part, int64_t pstride, int* err_flag) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, nthr = blockDim.x;
  const int m = P.m, mv = P.mv, qv = P.qv, d = P.d, dv = P.dv;
  float* p = sm;
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

  for (int i = tid; i < mv * qv; i += nthr) Zc[i] = P.zc[i];

  const int MT = (m + 3) >> 2;
  const int64_t units = int64_t(MT) * (MT + 1) / 2;
  const int64_t u0 = units * warp / nw, u1 = units * (warp + 1) / nw;
  int at0 = 0, bt0 = 0;
  {
    int64_t start = 0;
    while (at0 < MT && start + (MT - at0) <= u0) {
      start += MT - at0;
      ++at0;
    }
    bt0 = at0 + int(u0 - start);
  }
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
    // psi1 values, stored [n][m] for the Psi tiles
    {
      float mu[Q], d1[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        mu[q] = R.mu[q * 32 + lane];
        d1[q] = R.d1[q * 32 + lane];
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
            e = fmaf(df * df, d1[q], e);
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

    // ---- psi2: upper-triangle 4x4 pair tiles, one datapoint per lane ----
    if (u0 < u1) {
      float kk[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) kk[q] = R.kk[q * 32 + lane];
      float w[4][Q], La[4];
      int at = at0, bt = bt0, cur = -1;
      for (int64_t u = u0; u < u1; ++u) {
        if (at != cur) {
          cur = at;
#pragma unroll
          for (int ai = 0; ai < 4; ++ai) {
            float z[Q];
            load_z<Q>(Zc + (4 * at + ai) * qv, z);
#pragma unroll
            for (int q = 0; q < Q; ++q) w[ai][q] = kk[q] * z[q];
            La[ai] = Ls[(4 * at + ai) * 32 + lane];
          }
        }
        float v[16];
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
          const int b = 4 * bt + bi;
          float zb[Q];
          load_z<Q>(Zc + b * qv, zb);
          const float Lb = Ls[b * 32 + lane];
#pragma unroll
          for (int ai = 0; ai < 4; ++ai) {
            float s = La[ai] + Lb;
#pragma unroll
            for (int q = 0; q < Q; ++q) s = fmaf(w[ai][q], zb[q], s);
            float e = ex2(s);
            if (at == bt && bi < ai) e = 0.f;
            v[ai * 4 + bi] = e;
          }
        }
        const float tot = reduce_scatter16(v, lane);
        if (!(lane & 1)) {
          const int k = lane >> 1;
          const int a = 4 * at + (k >> 2), b = 4 * bt + (k & 3);
          if (b < m && a <= b) atomicAdd(phi_part + pair_index(a, b, m), double(tot));
        }
        if (++bt == MT) {
          ++at;
          bt = at;
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
        const float va[4] = {vv.x, vv.y, vv.z, vv.w}, ya[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(va[i], ya[j], acc[i][j]);
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
  // fixed-order CTA reduction of the scalar partials
  yy_acc = warp_sum_d(yy_acc);
  kl_acc = warp_sum_d(kl_acc);
  if (lane == 0) {
    red[warp] = yy_acc;
    red[32 + warp] = kl_acc;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < nw; ++i) {
      a += red[i];
      b += red[32 + i];
    }
    cta_part[0] = a;
    cta_part[1] = b;
  }
}

// =============================================================================
// Backward: global-gradient partials (d_variance, d_lengthscales, d_z) per CTA
// and the per-datapoint d_mu / d_s (written directly).
// =============================================================================
template <int Q>
__global__ void __launch_bounds__(512)
    psi_bwd_kernel(PsiConst P, BwdConst B, int64_t nchunks, double* __restrict__ part, int64_t pstride) {
  constexpr int NACC = 2 + 5 * Q;
  constexpr int T0 = 0, Y1 = 1, Y2 = 1 + Q, XX = 1 + 2 * Q, P0 = 1 + 3 * Q, P1 = 2 + 3 * Q, P2 = 2 + 4 * Q;
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, nthr = blockDim.x;
  const int m = P.m, mv = P.mv, qv = P.qv, d = P.d;
  float* p = sm;
  float* Zc = p;
  p += mv * qv;
  Rows R = carve_rows(p, qv);
  float* Ls = p;
  p += mv * 32;
  float* Ys = p;
  p += P.dv * 32;
  float* G1s = p;
  p += mv * 32;
  float* acc = p;
  p += nw * NACC * 32;
  double* dacc = reinterpret_cast<double*>(p);  // [(Q+1)][32]: d_lengthscales per (q, lane), d_variance

  for (int i = tid; i < mv * qv; i += nthr) Zc[i] = P.zc[i];
  for (int i = tid; i < (Q + 1) * 32; i += nthr) dacc[i] = 0.0;

  const int MT = (m + 3) >> 2;
  double* const cta_part = part + int64_t(blockIdx.x) * pstride;
  double* const dz_part = cta_part + 1 + P.q;
  const double inv_var = 1.0 / P.variance_d;

  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int64_t n0 = chunk * 32, n = n0 + lane;
    const bool valid = n < P.n;
    load_rows<Q>(P, n0, R, nullptr, nullptr);
    build_L<Q>(P, R, Zc, Ls);
    for (int dd = warp; dd < d; dd += nw) Ys[dd * 32 + lane] = valid ? float(P.y[dd * P.ld_y + n]) : 0.f;
    for (int i = tid; i < nw * NACC * 32; i += nthr) acc[i] = 0.f;
    __syncthreads();
    // psi1 adjoint weights G1_nm = v1_nm * <y_n, dPsi_m>
    {
      float mu[Q], d1[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        mu[q] = R.mu[q * 32 + lane];
        d1[q] = R.d1[q * 32 + lane];
      }
      const float b1 = R.b1[lane];
      for (int mt = warp; mt < (mv >> 2); mt += nw) {
        float w4[4] = {0.f, 0.f, 0.f, 0.f};
        for (int dd = 0; dd < d; ++dd) {
          const float yv = Ys[dd * 32 + lane];
          const float4 dp = __ldg(reinterpret_cast<const float4*>(B.dpsi + int64_t(dd) * mv) + mt);
          w4[0] = fmaf(yv, dp.x, w4[0]);
          w4[1] = fmaf(yv, dp.y, w4[1]);
          w4[2] = fmaf(yv, dp.z, w4[2]);
          w4[3] = fmaf(yv, dp.w, w4[3]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int mm = 4 * mt + i;
          float g = 0.f;
          if (mm < m) {
            float z[Q];
            load_z<Q>(Zc + mm * qv, z);
            float e = 0.f;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              const float df = mu[q] - z[q];
              e = fmaf(df * df, d1[q], e);
            }
            g = w4[i] * ex2(fmaf(-0.5f * kLog2e, e, b1));
          }
          G1s[mm * 32 + lane] = g;
        }
      }
    }
    __syncthreads();

    // ---- psi2 + psi1 contractions; warp owns inducing tiles at = warp + k*nw ----
    {
      float* accw = acc + warp * NACC * 32;
      for (int at = warp; at < MT; at += nw) {
        float w[4][Q], La[4], Ra[4], S[4][Q];
        {
          float kk[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) kk[q] = R.kk[q * 32 + lane];
#pragma unroll
          for (int ai = 0; ai < 4; ++ai) {
            float z[Q];
            load_z<Q>(Zc + (4 * at + ai) * qv, z);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              w[ai][q] = kk[q] * z[q];
              S[ai][q] = 0.f;
            }
            La[ai] = Ls[(4 * at + ai) * 32 + lane];
            Ra[ai] = 0.f;
          }
        }
        const float* Ub = B.u + 4 * at;
#pragma unroll 2
        for (int b = 0; b < m; ++b) {
          float zb[Q];
          load_z<Q>(Zc + b * qv, zb);
          const float Lb = Ls[b * 32 + lane];
          const float4 u4 = __ldg(reinterpret_cast<const float4*>(Ub + int64_t(b) * mv));
          const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
          for (int ai = 0; ai < 4; ++ai) {
            float s = La[ai] + Lb;
#pragma unroll
            for (int q = 0; q < Q; ++q) s = fmaf(w[ai][q], zb[q], s);
            const float g = uu[ai] * ex2(s);
            Ra[ai] += g;
#pragma unroll
            for (int q = 0; q < Q; ++q) S[ai][q] = fmaf(g, zb[q], S[ai][q]);
          }
        }
        // psi1 weights of the same inducing indices
        float g1[4];
#pragma unroll
        for (int ai = 0; ai < 4; ++ai) g1[ai] = G1s[(4 * at + ai) * 32 + lane];
        // per-datapoint contractions (lane-private rows of the warp's accumulator)
        {
          float t0 = 0.f, p0 = 0.f;
#pragma unroll
          for (int ai = 0; ai < 4; ++ai) {
            t0 += Ra[ai];
            p0 += g1[ai];
          }
          accw[T0 * 32 + lane] += t0;
          accw[P0 * 32 + lane] += p0;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            float y1 = 0.f, y2 = 0.f, xq = 0.f, p1 = 0.f, p2 = 0.f;
#pragma unroll
            for (int ai = 0; ai < 4; ++ai) {
              const float z = Zc[(4 * at + ai) * qv + q];
              y1 = fmaf(z, Ra[ai], y1);
              y2 = fmaf(z * z, Ra[ai], y2);
              xq = fmaf(z, S[ai][q], xq);
              p1 = fmaf(z, g1[ai], p1);
              p2 = fmaf(z * z, g1[ai], p2);
            }
            accw[(Y1 + q) * 32 + lane] += y1;
            accw[(Y2 + q) * 32 + lane] += y2;
            accw[(XX + q) * 32 + lane] += xq;
            accw[(P1 + q) * 32 + lane] += p1;
            accw[(P2 + q) * 32 + lane] += p2;
          }
        }
        // per-inducing contractions: d_z contribution of this datapoint (natural-log units)
        constexpr int K = 4 * Q, NG = (K + 31) / 32;
        float vals[NG * 32];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const float mu = R.mu[q * 32 + lane], d2 = R.d2[q * 32 + lane], d1 = R.d1[q * 32 + lane];
          const float kn = R.sv[q * 32 + lane] * P.il2[q] * d2;  // (1/l^2 - d2)/2
          const float c2 = 0.5f * (P.il2[q] + d2);
#pragma unroll
          for (int ai = 0; ai < 4; ++ai) {
            const float z = Zc[(4 * at + ai) * qv + q];
            const float v2 = 2.f * (fmaf(d2, mu, -c2 * z) * Ra[ai] + kn * S[ai][q]);
            const float v1 = g1[ai] * d1 * (mu - z);
            vals[ai * Q + q] = v2 + v1;
          }
        }
#pragma unroll
        for (int i = K; i < NG * 32; ++i) vals[i] = 0.f;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          float v32[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v32[i] = vals[g * 32 + i];
          const float tot = reduce_scatter32(v32, lane);
          const int idx = g * 32 + lane;
          if (idx < K) {
            const int ai = idx / Q, q = idx - ai * Q, a = 4 * at + ai;
            if (a < m && q < P.q) atomicAdd(dz_part + a + int64_t(q) * m, double(tot));
          }
        }
      }
    }
    __syncthreads();

    // ---- per-datapoint epilogue: d_mu, d_s and the d_lengthscales / d_variance shares ----
    for (int q = warp; q < P.q; q += nw) {
      if (!valid) continue;
      double t0 = 0, y1 = 0, y2 = 0, xq = 0, p0 = 0, p1 = 0, p2 = 0;
      for (int w2 = 0; w2 < nw; ++w2) {
        const float* a = acc + w2 * NACC * 32;
        t0 += a[T0 * 32 + lane];
        y1 += a[(Y1 + q) * 32 + lane];
        y2 += a[(Y2 + q) * 32 + lane];
        xq += a[(XX + q) * 32 + lane];
        p0 += a[P0 * 32 + lane];
        p1 += a[(P1 + q) * 32 + lane];
        p2 += a[(P2 + q) * 32 + lane];
      }
      const double mu = R.mu[q * 32 + lane], sv = R.sv[q * 32 + lane];
      const double l = P.ls[q], l2 = l * l, il2 = 1.0 / l2, il3 = il2 / l;
      const double d2 = 1.0 / (2.0 * sv + l2), d1 = 1.0 / (sv + l2);
      const double q1 = mu * mu * p0 - 2.0 * mu * p1 + p2;  // sum_m G1 (mu - z_m)^2
      const double dl = t0 * (2.0 * sv * d2 / l + 2.0 * l * d2 * d2 * mu * mu) - 4.0 * l * d2 * d2 * mu * y1 +
                        y2 * (il3 + l * d2 * d2) - xq * (il3 - l * d2 * d2) + sv * d1 * p0 / l +
                        l * d1 * d1 * q1;
      dacc[q * 32 + lane] += dl;
      if (q == 0) dacc[Q * 32 + lane] += (2.0 * t0 + p0) * inv_var;
      if (B.write_local) {
        double dmu = -2.0 * d2 * mu * t0 + 2.0 * d2 * y1 - d1 * (mu * p0 - p1);
        double ds = t0 * (-d2 + 2.0 * d2 * d2 * mu * mu) - 4.0 * d2 * d2 * mu * y1 + d2 * d2 * (y2 + xq) -
                    0.5 * d1 * p0 + 0.5 * d1 * d1 * q1;
        if (B.add_kl) {
          const double mo = P.mu[q * P.ld_mu + n], so = P.s[q * P.ld_s + n];
          dmu -= mo;
          ds -= 0.5 * (1.0 - 1.0 / so);
        }
        B.d_mu[q * B.ld_g + n] = dmu;
        B.d_s[q * B.ld_g + n] = ds;
      }
    }
    __syncthreads();
  }
  if (tid <= Q) {
    double s = 0.0;
    for (int l = 0; l < 32; ++l) s += dacc[tid * 32 + l];
    if (tid < P.q)
      cta_part[1 + tid] = s;
    else if (tid == Q)
      cta_part[0] = s;
  }
}

// Fixed-order column sums of nparts partial rows: a block covers 32 columns with 8 warps, warp w
// summing rows w, w + 8, ... (coalesced across the columns), then the 8 partial sums in order.
// Launch with 256 threads and ceil(count / 32) blocks.
__device__ __forceinline__ bool colsum8(const double* __restrict__ part, int64_t pstride, int nparts, int64_t count,
                                        int64_t& k, double& sum) {
  __shared__ double red[8][32];
  const int kk = threadIdx.x & 31, w = threadIdx.x >> 5;
  k = int64_t(blockIdx.x) * 32 + kk;
  double s = 0.0;
  if (k < count)
    for (int c = w; c < nparts; c += 8) s += part[c * pstride + k];
  red[w][kk] = s;
  __syncthreads();
  if (w != 0 || k >= count) return false;
  sum = red[0][kk];
  for (int i = 1; i < 8; ++i) sum += red[i][kk];
  return true;
}

// Fixed-order reduction of the per-CTA forward partials into the packed stats vector.
__global__ void __launch_bounds__(256) fwd_reduce_kernel(const double* __restrict__ part, int64_t pstride, int nparts,
                                                         int64_t count, double* __restrict__ packed, double phi_val,
                                                         double n_count) {
  int64_t k;
  double s;
  if (colsum8(part, pstride, nparts, count, k, s)) {
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

__global__ void __launch_bounds__(256) bwd_reduce_kernel(const double* __restrict__ part, int64_t pstride, int nparts,
                                                         int64_t count, double* __restrict__ packed, double dvar0) {
  int64_t k;
  double s;
  if (colsum8(part, pstride, nparts, count, k, s)) packed[k] = (k == 0 ? dvar0 : 0.0) + s;
}

template <int Q>
__global__ void psi1_matrix_kernel(PsiConst P, double* __restrict__ out, int64_t ld_out) {
  const int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int mm = blockIdx.y;
  if (n >= P.n || mm >= P.m) return;
  double e = 0.0, lc = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (q >= P.q) break;
    const double mu = P.mu[q * P.ld_mu + n], s = P.s[q * P.ld_s + n];
    const double l2 = P.ls[q] * P.ls[q];
    const double df = mu - P.z64[mm + int64_t(q) * P.m];
    e += df * df / (s + l2);
    lc += log1p(s / l2);
  }
  out[mm * ld_out + n] = P.variance_d * exp(-0.5 * lc - 0.5 * e);
}

// ---------------------------------------------------------------------------
// Host-side dispatch over the instantiated latent dimensions.
// ---------------------------------------------------------------------------
constexpr int kQs[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32};

int pick_q(int q) {
  for (int v : kQs)
    if (v >= q) return v;
  return -1;
}

int choose_bwd_warps(int mt) {
  if (mt <= 4) return mt < 1 ? 1 : mt;
  int best = 4;
  double best_eff = 0.0;
  for (int nw = 4; nw <= 16; ++nw) {
    const int per = (mt + nw - 1) / nw;
    const double eff = double(mt) / double(per * nw);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = nw;
    }
  }
  return best;
}

size_t fwd_smem(const PsiConst& P) {
  return sizeof(float) * (size_t(P.mv) * P.qv + rows_floats(P.qv) + size_t(P.mv) * 32 * 2 + 32 * size_t(P.dv)) +
         64 * sizeof(double);
}

size_t bwd_smem(const PsiConst& P, int nw, int Q) {
  return sizeof(float) * (size_t(P.mv) * P.qv + rows_floats(P.qv) + size_t(P.mv) * 32 * 2 + size_t(P.dv) * 32 +
                          size_t(nw) * (2 + 5 * Q) * 32) +
         (Q + 1) * 32 * sizeof(double);
}

template <int Q>
int plan_fwd_q(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  const int64_t nchunks = (P.n + 31) / 32;
  const int threads = 256;
  const size_t smem = fwd_smem(P);
  auto kern = psi_fwd_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) return 3;
  *geom = LaunchGeom{int(std::min<int64_t>(nchunks, int64_t(num_sms) * occ)), threads, smem};
  return 0;
}

template <int Q>
int plan_bwd_q(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  const int64_t nchunks = (P.n + 31) / 32;
  int nw = choose_bwd_warps((P.m + 3) / 4);
  while (nw > 1 && bwd_smem(P, nw, Q) > 227 * 1024) nw = (nw + 1) / 2;
  const int threads = 32 * nw;
  const size_t smem = bwd_smem(P, nw, Q);
  auto kern = psi_bwd_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) return 3;
  *geom = LaunchGeom{int(std::min<int64_t>(nchunks, int64_t(num_sms) * occ)), threads, smem};
  return 0;
}

template <int Q>
int launch_fwd(const PsiConst& P, double* part, double* packed, int* err_flag, int num_sms, cudaStream_t st,
               LaunchGeom* geom, cudaEvent_t e0, cudaEvent_t e1) {
  LaunchGeom g{};
  if (int rc = plan_fwd_q<Q>(P, num_sms, &g)) return rc;
  const int64_t nchunks = (P.n + 31) / 32;
  const int64_t pstride = fwd_part_count(P.m, P.d);
  if (g.grid > 0) {
    if (cudaMemsetAsync(part, 0, sizeof(double) * pstride * g.grid, st) != cudaSuccess) return 3;
    if (e0) cudaEventRecord(e0, st);
    psi_fwd_kernel<Q><<<g.grid, g.threads, g.smem, st>>>(P, nchunks, part, pstride, err_flag);
    if (e1) cudaEventRecord(e1, st);
    g_launches.fetch_add(1);
  }
  fwd_reduce_kernel<<<int((pstride + 31) / 32), 256, 0, st>>>(part, pstride, g.grid, pstride, packed,
                                                                 double(P.n) * P.variance_d, double(P.n));
  g_launches.fetch_add(1);
  if (geom) *geom = g;
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int Q>
int launch_bwd(const PsiConst& P, const BwdConst& B, double* part, double* packed, int num_sms, cudaStream_t st,
               LaunchGeom* geom, cudaEvent_t e0, cudaEvent_t e1) {
  LaunchGeom g{};
  if (int rc = plan_bwd_q<Q>(P, num_sms, &g)) return rc;
  const int64_t nchunks = (P.n + 31) / 32;
  const int64_t pstride = bwd_part_count(P.m, P.q);
  if (g.grid > 0) {
    if (cudaMemsetAsync(part, 0, sizeof(double) * pstride * g.grid, st) != cudaSuccess) return 3;
    if (e0) cudaEventRecord(e0, st);
    psi_bwd_kernel<Q><<<g.grid, g.threads, g.smem, st>>>(P, B, nchunks, part, pstride);
    if (e1) cudaEventRecord(e1, st);
    g_launches.fetch_add(1);
  }
  bwd_reduce_kernel<<<int((pstride + 31) / 32), 256, 0, st>>>(part, pstride, g.grid, pstride, packed,
                                                                 B.d_phi * double(P.n));
  g_launches.fetch_add(1);
  if (geom) *geom = g;
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

extern std::atomic<int64_t> g_tc_launches;
int64_t launches_issued() { return g_launches.load() + g_tc_launches.load(); }

// Kernel family: tensor-core (tcgen05) psi2 when the shape fits (M <= 128), else SIMT.
// SGPX_PSI_IMPL=simt forces the SIMT kernels (A/B comparisons, profiling).
int impl_forced() {
  static const int forced = [] {
    const char* e = getenv("SGPX_PSI_IMPL");
    if (!e) return 0;
    if (!strcmp(e, "simt")) return 1;
    if (!strcmp(e, "tc")) return 2;
    return 0;
  }();
  return forced;
}

// Row-tile tensor-core psi2: the default where it fits; SGPX_PSI_IMPL=simt|tc selects the older
// kernels.  The deterministic (SGPR) kernel is narrower (den = 1/l^2, no 2S), so its pairs with
// weight sit closer to z-bar and the assembly from the exponent-as-GEMM sums cancels harder: it runs
// in the precise mode (rt_pieces) and only up to Q = 16 (d_l <= 2.1e-5) — beyond that d_l from the
// backward sums exceeds the 5e-5 tolerance (6e-5 .. 9e-5 at Q = 18 / 20), and the direct-difference
// kernels run (tools/dbg_q.py, profiles/accuracy/r01_q_sweep_*.log).  SGPX_RT_DET=0|1 overrides (A/B).
bool use_rt(const PsiConst& P) {
  static const int det = [] {
    const char* e = getenv("SGPX_RT_DET");
    return e ? (atoi(e) != 0 ? 1 : 0) : -1;
  }();
  const bool det_ok = det < 0 ? instantiated_q(P.q) <= 16 : det == 1;
  return impl_forced() == 0 && (P.expected || det_ok) && rt_supported(P);
}

const double* rt_fwd_region(const PsiConst& P, const double* fwd_part, int num_sms) {
  return fwd_part + int64_t(psi1_fwd_rows(P, num_sms)) * fwd_part_count(P.m, P.d);
}

bool use_tc(const PsiConst& P, bool backward) {
  const int forced = impl_forced();
  if (forced == 1) return false;
  if (backward) return tc_backward_available() && tc_backward_fits(P);
  // forward: the SIMT kernel is faster until the TC forward is restructured (profiles/r01_*)
  return forced == 2 && tc_supported(P);
}

int instantiated_q(int q) { return pick_q(q); }

#define SGPX_DISPATCH_Q(QV, CALL)   \
  switch (QV) {                     \
    case 1: return CALL(1);         \
    case 2: return CALL(2);         \
    case 3: return CALL(3);         \
    case 4: return CALL(4);         \
    case 5: return CALL(5);         \
    case 6: return CALL(6);         \
    case 8: return CALL(8);         \
    case 10: return CALL(10);       \
    case 12: return CALL(12);       \
    case 16: return CALL(16);       \
    case 20: return CALL(20);       \
    case 24: return CALL(24);       \
    case 32: return CALL(32);       \
    default: return 1;              \
  }

int psi_forward(const PsiConst& P, double* part, double* packed, int* err_flag, int num_sms, void* stream,
                LaunchGeom* geom, void* ev_begin, void* ev_end) {
  if (use_rt(P)) {
    LaunchGeom g{};
    if (int rc = plan_forward(P, num_sms, &g)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t pstride = fwd_part_count(P.m, P.d);
    const int g1 = psi1_fwd_rows(P, num_sms);
    if (g1 > 0 && cudaMemsetAsync(part, 0, sizeof(double) * pstride * g1, st) != cudaSuccess) return 3;
    if (ev_begin) cudaEventRecord(cudaEvent_t(ev_begin), st);
    if (g1 > 0) {
      if (int rc = psi1_forward(P, part, pstride, g1, err_flag, stream, 1)) return rc;
    }
    fwd_reduce_kernel<<<int((pstride + 31) / 32), 256, 0, st>>>(part, pstride, g1, pstride, packed,
                                                                   double(P.n) * P.variance_d, double(P.n));
    g_launches.fetch_add(1);
    if (int rc = rt_forward(P, part + int64_t(g1) * pstride, packed, num_sms, stream)) return rc;
    if (ev_end) cudaEventRecord(cudaEvent_t(ev_end), st);
    if (geom) *geom = g;
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  if (use_tc(P, false)) return psi_forward_tc(P, part, packed, err_flag, num_sms, stream, geom, ev_begin, ev_end);
  const int qi = pick_q(P.q);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define CALL_FWD(QQ) \
  launch_fwd<QQ>(P, part, packed, err_flag, num_sms, st, geom, cudaEvent_t(ev_begin), cudaEvent_t(ev_end))
  SGPX_DISPATCH_Q(qi, CALL_FWD)
#undef CALL_FWD
}

int psi_backward(const PsiConst& P, const BwdConst& B, double* part, double* packed, int num_sms, void* stream,
                 LaunchGeom* geom, void* ev_begin, void* ev_end) {
  if (use_rt(P)) {
    if (!B.fwd_rt) return 1;
    LaunchGeom g{};
    if (int rc = plan_backward(P, num_sms, &g)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t pstride = bwd_part_count(P.m, P.q);
    const int r1 = P.n > 0 ? psi1_bwd_rows(P, num_sms) : 0, rows = r1 + 1;
    if (cudaMemsetAsync(part, 0, sizeof(double) * pstride * rows, st) != cudaSuccess) return 3;
    if (ev_begin) cudaEventRecord(cudaEvent_t(ev_begin), st);
    // psi1 first: it writes d_mu / d_s (psi1 + KL parts); the psi2 kernel accumulates into them
    if (r1 > 0) {
      if (int rc = psi1_backward(P, B, part, pstride, r1, stream)) return rc;
    }
    if (int rc = rt_backward(P, B, part + int64_t(rows) * pstride, part + int64_t(r1) * pstride, num_sms, stream))
      return rc;
    if (ev_end) cudaEventRecord(cudaEvent_t(ev_end), st);
    const int64_t rt_rows = (rt_bwd_doubles(P, num_sms) + pstride - 1) / pstride;
    double* tmp = part + (int64_t(rows) + rt_rows) * pstride;
    if (int rc = bwd_reduce_rows(part, pstride, rows, packed, B.d_phi * double(P.n), tmp, stream)) return rc;
    if (geom) *geom = g;
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  if (use_tc(P, true)) return psi_backward_tc(P, B, part, packed, num_sms, stream, geom, ev_begin, ev_end);
  const int qi = pick_q(P.q);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define CALL_BWD(QQ) \
  launch_bwd<QQ>(P, B, part, packed, num_sms, st, geom, cudaEvent_t(ev_begin), cudaEvent_t(ev_end))
  SGPX_DISPATCH_Q(qi, CALL_BWD)
#undef CALL_BWD
}

int plan_forward(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  if (use_rt(P)) {  // partial rows: psi1 rows + the row-tile region
    const int64_t pstride = fwd_part_count(P.m, P.d);
    const int64_t extra = (rt_fwd_doubles(P, num_sms) + pstride - 1) / pstride;
    *geom = LaunchGeom{int(psi1_fwd_rows(P, num_sms) + extra), 448, 0};
    return 0;
  }
  if (use_tc(P, false)) return plan_forward_tc(P, num_sms, geom);
  const int qi = pick_q(P.q);
#define CALL_PF(QQ) plan_fwd_q<QQ>(P, num_sms, geom)
  SGPX_DISPATCH_Q(qi, CALL_PF)
#undef CALL_PF
}

int plan_backward(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  if (use_rt(P)) {  // psi1 rows (8 per CTA) + 1 psi2 row + the row-tile scratch
    const int64_t pstride = bwd_part_count(P.m, P.q);
    const int r1 = P.n > 0 ? psi1_bwd_rows(P, num_sms) : 0;
    const int64_t extra = (rt_bwd_doubles(P, num_sms) + pstride - 1) / pstride +
                          (bwd_reduce_tmp_doubles(pstride) + pstride - 1) / pstride;
    *geom = LaunchGeom{int(r1 + 1 + extra), 448, 0};
    return 0;
  }
  if (use_tc(P, true)) return plan_backward_tc(P, num_sms, geom);
  const int qi = pick_q(P.q);
#define CALL_PB(QQ) plan_bwd_q<QQ>(P, num_sms, geom)
  SGPX_DISPATCH_Q(qi, CALL_PB)
#undef CALL_PB
}

int psi1_matrix(const PsiConst& P, double* out, int64_t ld_out, void* stream) {
  const int qi = pick_q(P.q);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (P.n == 0 || P.m == 0) return 0;
  dim3 grid(unsigned((P.n + 127) / 128), unsigned(P.m));
#define CALL_P1(QQ) (psi1_matrix_kernel<QQ><<<grid, 128, 0, st>>>(P, out, ld_out), g_launches.fetch_add(1), \
                     cudaGetLastError() == cudaSuccess ? 0 : 3)
  SGPX_DISPATCH_Q(qi, CALL_P1)
#undef CALL_P1
}

}  // namespace sgpx
