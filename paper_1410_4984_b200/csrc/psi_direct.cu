// psi_direct.cu -- direct-difference psi-statistics kernels: the accurate path.
//
// Reference: psi_stats.hpp:144-326 (detail::sweep_stats), both modes.  These kernels evaluate
// every exponent in the reference's own direct-difference form, in fp64:
//   psi1  e1 = sum_q (mu_q - z_mq)^2 / (S_q + l_q^2)           (psi_stats.hpp:176-183)
//   psi2  e2 = sum_q (mu_q - zbar_q)^2 / (2 S_q + l_q^2)        (psi_stats.hpp:258-263)
// (the deterministic mode is the S = 0 case: c1 = var, c2 = var^2, den = 1/l^2, and
// 1/2 sum((x-za)^2 + (x-zb)^2)/l^2 = sum (x-zbar)^2/l^2 + sum (za-zb)^2/(4 l^2), :264-271), then
// v = 2^(log2 c + log2 pconst - log2e e) in fp64 (exp2_d, ~1 ulp).  No expansion of (mu - zbar)^2 is
// formed and no step is below fp64, so the
// accuracy does not depend on how far mu and Z sit from each other or from any centre: this is
// the path the engine routes to when the inducing points spread beyond the tensor-core path's
// measured envelope, and for latent dimensions without a row-tile instantiation.
//
// Work split (every cross-thread / cross-CTA sum in a fixed order, no atomics):
//   forward   dir_pair_fwd_kernel   thread per pair p = (a <= b), datapoints streamed through
//                                   shared memory: Phi_p = sum_n v and R_pq = sum_n v rb_q,
//                                   rb = d2 (mu - zbar) (the U-independent pair sums of the
//                                   gradient, kept for the backward)
//             dir_psi1_fwd_kernel   32 inducing points x 64 output columns per CTA:
//                                   Psi_md = sum_n v1_nm y_nd
//             dir_rows_kernel       yy, KL partials, validation flags
//   backward  dla::gemm             W = Y dPsi^T (fp64), the psi1 adjoint weights w_nm = <y_n, dPsi_m>
//             dir_psi1_bwd_kernel   thread per datapoint: uv = w v1, the psi1
//                                   parts of d mu, d S (+ KL), d l, d var; d Z_m by warp trees
//             dir_pair_bwd_kernel   thread per datapoint: T0 = sum_p uv, A_q = sum_p uv diff_q,
//                                   C_q = sum_p uv diff_q^2  ->  d mu -= 2 d2 A, d S += d2 (2 d2 C - T0),
//                                   d l += 2 l d2^2 C + 2 S d2 / l T0
//             dir_pair_dz/dl        the per-pair terms from (Phi_p, R_pq) and the adjoint weights
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <atomic>

#include "dla.cuh"
#include "psi_common.cuh"
#include "psi_kernels.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;

namespace {
using namespace dev;

constexpr int kCh = 32;          // datapoints staged per chunk (forward sweeps)
constexpr int kPairThreads = 128;
constexpr double kLog2eD = 1.4426950408889634;

// 2^x in fp64: x = j + f with j = rint(x), |f| <= 1/2; 2^f = e^(f ln 2) by a degree-13 Taylor
// polynomial in Horner form (truncation < 2^-60 for |f ln 2| <= 0.35), times the exact 2^j.
// ~1 ulp, the accuracy of the reference's std::exp; underflows to exactly 0 below 2^-1020.
__device__ __forceinline__ double exp2_d(double x) {
  if (!(x > -1020.0)) return 0.0;  // also -inf: exactly 0
  const double j = rint(x);
  const double t = (x - j) * 0.69314718055994530942;
  double p = 1.0 / 6227020800.0;  // 1/13!
  p = fma(p, t, 1.0 / 479001600.0);
  p = fma(p, t, 1.0 / 39916800.0);
  p = fma(p, t, 1.0 / 3628800.0);
  p = fma(p, t, 1.0 / 362880.0);
  p = fma(p, t, 1.0 / 40320.0);
  p = fma(p, t, 1.0 / 5040.0);
  p = fma(p, t, 1.0 / 720.0);
  p = fma(p, t, 1.0 / 120.0);
  p = fma(p, t, 1.0 / 24.0);
  p = fma(p, t, 1.0 / 6.0);
  p = fma(p, t, 0.5);
  p = fma(p, t, 1.0);
  p = fma(p, t, 1.0);
  return p * __hiloint2double((int(j) + 1023) << 20, 0);
}

__device__ __forceinline__ void pair_of(int64_t p, int m, int& a, int& b) {
  // m1-major upper triangle (psi_stats.hpp:85-97): rows of length m, m-1, ...
  const double t = 2.0 * m + 1.0;
  int x = int((t - sqrt(t * t - 8.0 * double(p))) * 0.5);
  x = x < 0 ? 0 : (x >= m ? m - 1 : x);
  auto start = [m](int r) { return int64_t(r) * m - int64_t(r) * (r - 1) / 2; };
  while (x + 1 < m && start(x + 1) <= p) ++x;
  while (x > 0 && start(x) > p) --x;
  a = x;
  b = int(p - start(x)) + x;
}

__device__ __forceinline__ double pair_weight(const double* u, int mv, int a, int b) {
  return a == b ? u[a * mv + a] : u[a * mv + b] + u[b * mv + a];
}

// log2 c2_n (psi2) or log2 c1_n (psi1) of datapoint n (psi_stats.hpp:148-163): fact = 2 or 1.
__device__ __forceinline__ double log2_c(const PsiConst& P, int64_t n, double fact, double powvar) {
  double lc = powvar;
  if (P.expected)
    for (int q = 0; q < P.q; ++q) {
      const double s = P.s[q * P.ld_s + n];
      lc -= 0.5 * log2(1.0 + fact * s / (P.ls[q] * P.ls[q]));
    }
  return lc;
}

// ---------------------------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(kPairThreads) dir_pair_fwd_kernel(PsiConst P, int64_t npairs, int64_t cps,
                                                                    double* __restrict__ part) {
  __shared__ double s_mu[Q][kCh], s_d2[Q][kCh], s_lc[kCh];
  const int tid = threadIdx.x;
  const int64_t p = int64_t(blockIdx.x) * kPairThreads + tid;
  const int m = P.m;
  double zb[Q], acc[Q], phi = 0.0, lp = 0.0;
  if (p < npairs) {
    int a, b;
    pair_of(p, m, a, b);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      zb[q] = 0.0;
      acc[q] = 0.0;
      if (q < P.q) {
        const double za = P.z64[q * m + a], zz = P.z64[q * m + b];
        zb[q] = 0.5 * (za + zz);
        const double dz = (za - zz) / P.ls[q];
        lp += dz * dz;
      }
    }
    lp *= -0.25 * kLog2eD;  // log2 pconst = -log2e sum (za - zb)^2 / (4 l^2)   (psi_stats.hpp:240-246)
  } else {
#pragma unroll
    for (int q = 0; q < Q; ++q) zb[q] = acc[q] = 0.0;
  }
  const int64_t nchunks = (P.n + kCh - 1) / kCh;
  const int64_t c0 = int64_t(blockIdx.y) * cps, c1 = min(nchunks, c0 + cps);
  const double lvar = 2.0 * log2(P.variance_d);
  for (int64_t c = c0; c < c1; ++c) {
    const int64_t n0 = c * kCh;
    __syncthreads();
    for (int i = tid; i < Q * kCh; i += kPairThreads) {
      const int q = i / kCh, j = i % kCh;
      const int64_t n = n0 + j;
      double mu = 0.0, d2 = 0.0;
      if (q < P.q && n < P.n) {
        mu = P.mu[q * P.ld_mu + n];
        const double s = P.expected ? P.s[q * P.ld_s + n] : 0.0;
        d2 = 1.0 / (2.0 * s + P.ls[q] * P.ls[q]);
      }
      s_mu[q][j] = mu;
      s_d2[q][j] = d2;
    }
    if (tid < kCh) {
      const int64_t n = n0 + tid;
      s_lc[tid] = n < P.n ? log2_c(P, n, 2.0, lvar) : -CUDART_INF;
    }
    __syncthreads();
    if (p < npairs) {
#pragma unroll 2
      for (int j = 0; j < kCh; ++j) {
        double t[Q], e = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const double df = s_mu[q][j] - zb[q];
          t[q] = s_d2[q][j] * df;
          e = fma(t[q], df, e);
        }
        const double v = exp2_d(s_lc[j] + lp - kLog2eD * e);
        phi += v;
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[q] = fma(v, t[q], acc[q]);
      }
    }
  }
  if (p < npairs) {
    double* o = part + (int64_t(blockIdx.y) * npairs + p) * (Q + 1);
    o[0] = phi;
#pragma unroll
    for (int q = 0; q < Q; ++q) o[1 + q] = acc[q];
  }
}

// sums[p][k] = sum_split part[split][p][k] (ascending split order); packed[4 + p] = Phi_p
__global__ void dir_pair_reduce_kernel(const double* __restrict__ part, int ns, int64_t npairs, int w,
                                       double* __restrict__ sums, double* __restrict__ packed) {
  const int64_t total = npairs * w;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < ns; ++k) s += part[k * total + i];
    sums[i] = s;
    if (i % w == 0) packed[4 + i / w] = s;
  }
}

// Psi partials: CTA (m block of 32, split, d block of 64); part[split][m + d M]
template <int Q>
__global__ void __launch_bounds__(256) dir_psi1_fwd_kernel(PsiConst P, int64_t rps, double* __restrict__ part) {
  constexpr int CH = Q < 32 ? kCh : kCh / 2;  // datapoints per staged chunk (static shared memory < 48 KB)
  __shared__ double s_z[Q][32], s_mu[Q][CH], s_d1[Q][CH], s_lc[CH], s_v[CH][33], s_y[64][CH + 1];
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int m = P.m, m0 = blockIdx.x * 32, d0 = blockIdx.z * 64;
  for (int i = tid; i < Q * 32; i += 256) {
    const int q = i / 32, a = m0 + i % 32;
    s_z[q][i % 32] = (q < P.q && a < m) ? P.z64[q * m + a] : 0.0;
  }
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;
  const int64_t r0 = int64_t(blockIdx.y) * rps, r1 = min(P.n, r0 + rps);  // this split's rows
  const double lvar = log2(P.variance_d);
  for (int64_t n0 = r0; n0 < r1; n0 += CH) {
    __syncthreads();
    for (int i = tid; i < Q * CH; i += 256) {
      const int q = i / CH, j = i % CH;
      const int64_t n = n0 + j;
      double mu = 0.0, d1 = 0.0;
      if (q < P.q && n < P.n) {
        mu = P.mu[q * P.ld_mu + n];
        const double s = P.expected ? P.s[q * P.ld_s + n] : 0.0;
        d1 = 1.0 / (s + P.ls[q] * P.ls[q]);
      }
      s_mu[q][j] = mu;
      s_d1[q][j] = d1;
    }
    for (int i = tid; i < 64 * CH; i += 256) {
      const int dd = i / CH, j = i % CH;
      const int64_t n = n0 + j;
      s_y[dd][j] = (d0 + dd < P.d && n < P.n) ? P.y[(d0 + dd) * P.ld_y + n] : 0.0;
    }
    if (tid < CH) {
      const int64_t n = n0 + tid;
      s_lc[tid] = n < P.n ? log2_c(P, n, 1.0, lvar) : -CUDART_INF;
    }
    __syncthreads();
    // v1[j][a] for the 32 x 32 tile: warp wp takes datapoints j = wp, wp + 8, ..., lane = a
    for (int j = wp; j < CH; j += 8) {
      double e = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double df = s_mu[q][j] - s_z[q][lane];
        e = fma(s_d1[q][j] * df, df, e);
      }
      s_v[j][lane] = (m0 + lane < m) ? exp2_d(s_lc[j] - 0.5 * kLog2eD * e) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int dd = wp + 8 * k;
      double a = acc[k];
#pragma unroll 8
      for (int j = 0; j < CH; ++j) a = fma(s_v[j][lane], s_y[dd][j], a);
      acc[k] = a;
    }
  }
  const int a = m0 + lane;
  if (a < m)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int dd = d0 + wp + 8 * k;
      if (dd < P.d) part[int64_t(blockIdx.y) * m * P.d + a + int64_t(dd) * m] = acc[k];
    }
}

// yy and KL partials per block (fixed-order block trees), validation flags (psi_stats.hpp:119-125,
// parallel.hpp:148-149)
__global__ void __launch_bounds__(256) dir_rows_kernel(PsiConst P, int with_kl, double* __restrict__ part,
                                                       int* __restrict__ err_flag) {
  __shared__ double ry[256], rk[256];
  double yy = 0.0, kl = 0.0;
  int flag = 0;
  for (int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; n < P.n; n += int64_t(gridDim.x) * blockDim.x) {
    for (int q = 0; q < P.q; ++q) {
      const double mu = P.mu[q * P.ld_mu + n];
      if (!isfinite(mu)) flag |= 1;
      if (P.expected) {
        const double s = P.s[q * P.ld_s + n];
        if (!(s > 0.0 && isfinite(s))) flag |= 4;
        if (with_kl) kl += 0.5 * (s + mu * mu - log(s) - 1.0);
      }
    }
    for (int d = 0; d < P.d; ++d) {
      const double y = P.y[d * P.ld_y + n];
      if (!isfinite(y)) flag |= 1;
      yy += y * y;
    }
  }
  if (flag) atomicOr(err_flag, flag);
  ry[threadIdx.x] = yy;
  rk[threadIdx.x] = kl;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      ry[threadIdx.x] += ry[threadIdx.x + w];
      rk[threadIdx.x] += rk[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = ry[0];
    part[2 * blockIdx.x + 1] = rk[0];
  }
}

// packed[0..3] = phi, yy, n, kl;  packed[4 + P + i] = Psi_i (sum of the psi1 splits)
__global__ void dir_fwd_final_kernel(PsiConst P, const double* __restrict__ rows, int nrb,
                                     const double* __restrict__ p1, int ns1, double* __restrict__ packed) {
  const int64_t npairs = int64_t(P.m) * (P.m + 1) / 2, md = int64_t(P.m) * P.d;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < md; i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < ns1; ++k) s += p1[k * md + i];
    packed[4 + npairs + i] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double yy = 0.0, kl = 0.0;
    for (int k = 0; k < nrb; ++k) {
      yy += rows[2 * k];
      kl += rows[2 * k + 1];
    }
    packed[0] = double(P.n) * P.variance_d;
    packed[1] = yy;
    packed[2] = double(P.n);
    packed[3] = kl;
  }
}

// ---------------------------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------------------------
// psi1 per datapoint (psi_stats.hpp:189-216): thread per datapoint of a 128-row tile, inducing
// points in blocks of 32 (Z and dPsi staged in shared memory).  Writes d mu / d S (psi1 part, KL
// gradients when add_kl: parallel.hpp:163-166; the psi2 kernel adds its part afterwards) and the
// per-CTA row [d var, d l (Q), d Z (a + q M)] (persistent CTAs, owner-thread accumulation).
constexpr int kBwdThreads = 128;

template <int Q>
__global__ void __launch_bounds__(kBwdThreads) dir_psi1_bwd_kernel(PsiConst P, BwdConst B, int64_t rstride,
                                                                   double* __restrict__ rows,
                                                                   const double* __restrict__ W) {
  constexpr int KG = Q <= 32 ? 8 : 4;    // inducing points per d Z reduction group
  __shared__ double s_z[Q][32];
  __shared__ double s_dz[kBwdThreads / 32][KG][Q];
  __shared__ double s_red[kBwdThreads];
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int m = P.m;
  double* row = rows + int64_t(blockIdx.x) * rstride;  // [dvar, dl (Q), dz (a + q M)]
  for (int64_t i = tid; i < rstride; i += kBwdThreads) row[i] = 0.0;
  double dvar = 0.0, dl[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) dl[q] = 0.0;
  const int64_t ntiles = (P.n + kBwdThreads - 1) / kBwdThreads;
  const double lvar = log2(P.variance_d), ivar = 1.0 / P.variance_d;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t n = tile * kBwdThreads + tid;
    const bool valid = n < P.n;
    const int64_t nn = valid ? n : 0;
    double mu[Q], sv[Q], d1[Q], gmu[Q], gs[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      mu[q] = sv[q] = d1[q] = gmu[q] = gs[q] = 0.0;
      if (q < P.q) {
        mu[q] = P.mu[q * P.ld_mu + nn];
        sv[q] = P.expected ? P.s[q * P.ld_s + nn] : 0.0;
        d1[q] = 1.0 / (sv[q] + P.ls[q] * P.ls[q]);
      }
    }
    const double lc = valid ? log2_c(P, nn, 1.0, lvar) : -CUDART_INF;
    for (int m0 = 0; m0 < m; m0 += 32) {
      __syncthreads();
      for (int i = tid; i < Q * 32; i += kBwdThreads) {
        const int q = i / 32, a = m0 + i % 32;
        s_z[q][i % 32] = (q < P.q && a < m) ? P.z64[q * m + a] : 0.0;
      }
      __syncthreads();
      const int na = min(32, m - m0);
      for (int k0 = 0; k0 < na; k0 += KG) {
        const int kn = min(KG, na - k0);
        for (int kk = 0; kk < kn; ++kk) {
          const int k = k0 + kk;
          double e = 0.0, r[Q], df[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            df[q] = mu[q] - s_z[q][k];
            r[q] = df[q] * d1[q];
            e = fma(r[q], df[q], e);
          }
          // w_na = <y_n, dPsi_a> (W = Y dPsi^T, fp64 GEMM before this kernel)
          const double uv = (valid ? W[n + int64_t(m0 + k) * P.n] : 0.0) * exp2_d(lc - 0.5 * kLog2eD * e);
          dvar += uv * ivar;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            if (P.expected) {
              gmu[q] -= uv * r[q];
              gs[q] += uv * 0.5 * d1[q] * (r[q] * df[q] - 1.0);
              dl[q] += uv * P.ls[q] * d1[q] * (sv[q] / (P.ls[q] * P.ls[q]) + df[q] * r[q]);
            } else {
              dl[q] += uv * df[q] * df[q] / (P.ls[q] * P.ls[q] * P.ls[q]);
            }
            double zq = uv * r[q];  // d Z_aq += sum_n uv r  (fixed shuffle tree, then warps in order)
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) zq += __shfl_down_sync(0xffffffffu, zq, o);
            if (lane == 0) s_dz[wp][kk][q] = zq;
          }
        }
        __syncthreads();
        for (int i = tid; i < kn * Q; i += kBwdThreads) {
          const int kk = i / Q, q = i % Q;
          if (q < P.q) {
            double s = 0.0;
#pragma unroll
            for (int w2 = 0; w2 < kBwdThreads / 32; ++w2) s += s_dz[w2][kk][q];
            row[1 + P.q + (m0 + k0 + kk) + int64_t(q) * m] += s;
          }
        }
        __syncthreads();
      }
    }
    if (valid && B.write_local) {
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (q < P.q) {
          double a = gmu[q], b = gs[q];
          if (B.add_kl) {
            a -= mu[q];
            b -= 0.5 * (1.0 - 1.0 / sv[q]);
          }
          B.d_mu[q * B.ld_g + n] = a;
          B.d_s[q * B.ld_g + n] = b;
        }
    }
  }
  // block sums of d var, d l (fixed tree)
  for (int k = 0; k <= P.q; ++k) {
    double v = dvar;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (k == q + 1) v = dl[q];
    __syncthreads();
    s_red[tid] = v;
    __syncthreads();
    for (int w2 = kBwdThreads / 2; w2 > 0; w2 >>= 1) {
      if (tid < w2) s_red[tid] += s_red[tid + w2];
      __syncthreads();
    }
    if (tid == 0) row[k] += s_red[0];
  }
}

// psi2 per datapoint (psi_stats.hpp:279-304 restated on per-datapoint sums over the pairs).
template <int Q>
__global__ void __launch_bounds__(kBwdThreads) dir_pair_bwd_kernel(PsiConst P, BwdConst B, int64_t npairs,
                                                                   double* __restrict__ dl_rows) {
  constexpr int PS = Q <= 32 ? kBwdThreads : kBwdThreads / 2;  // pairs staged per step
  __shared__ double s_zb[Q][PS], s_lp[PS], s_w[PS];
  __shared__ double s_red[kBwdThreads];
  const int tid = threadIdx.x;
  const int m = P.m, mv = P.mv;
  double dl[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) dl[q] = 0.0;
  const int64_t ntiles = (P.n + kBwdThreads - 1) / kBwdThreads;
  const double lvar = 2.0 * log2(P.variance_d);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t n = tile * kBwdThreads + tid;
    const bool valid = n < P.n;
    const int64_t nn = valid ? n : 0;
    double mu[Q], d2[Q], sv[Q], A[Q], C[Q], T0 = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      mu[q] = d2[q] = sv[q] = A[q] = C[q] = 0.0;
      if (q < P.q) {
        mu[q] = P.mu[q * P.ld_mu + nn];
        sv[q] = P.expected ? P.s[q * P.ld_s + nn] : 0.0;
        d2[q] = 1.0 / (2.0 * sv[q] + P.ls[q] * P.ls[q]);
      }
    }
    const double lc = valid ? log2_c(P, nn, 2.0, lvar) : -CUDART_INF;
    for (int64_t p0 = 0; p0 < npairs; p0 += PS) {
      __syncthreads();
      if (tid < PS) {
        const int64_t p = p0 + tid;
        double lp = 0.0, w = 0.0;
        if (p < npairs) {
          int a, b;
          pair_of(p, m, a, b);
          w = pair_weight(B.u64, mv, a, b);
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            double zb = 0.0;
            if (q < P.q) {
              const double za = P.z64[q * m + a], zz = P.z64[q * m + b];
              zb = 0.5 * (za + zz);
              const double dz = (za - zz) / P.ls[q];
              lp += dz * dz;
            }
            s_zb[q][tid] = zb;
          }
          lp *= -0.25 * kLog2eD;
        } else {
#pragma unroll
          for (int q = 0; q < Q; ++q) s_zb[q][tid] = 0.0;
          lp = -CUDART_INF;
        }
        s_lp[tid] = lp;
        s_w[tid] = w;
      }
      __syncthreads();
      const int np = int(npairs - p0 < PS ? npairs - p0 : int64_t(PS));
#pragma unroll 2
      for (int k = 0; k < np; ++k) {
        double df[Q], e = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          df[q] = mu[q] - s_zb[q][k];
          e = fma(d2[q] * df[q], df[q], e);
        }
        const double uv = s_w[k] * exp2_d(lc + s_lp[k] - kLog2eD * e);
        T0 += uv;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const double t = uv * df[q];
          A[q] += t;
          C[q] = fma(t, df[q], C[q]);
        }
      }
    }
    if (valid) {
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (q < P.q) {
          const double l = P.ls[q];
          if (B.write_local) {
            B.d_mu[q * B.ld_g + n] += -2.0 * d2[q] * A[q];
            if (P.expected) B.d_s[q * B.ld_g + n] += d2[q] * (2.0 * d2[q] * C[q] - T0);
          }
          dl[q] += 2.0 * l * d2[q] * d2[q] * C[q] + 2.0 * sv[q] * d2[q] / l * T0;
        }
    }
  }
  for (int k = 0; k < P.q; ++k) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (k == q) v = dl[q];
    __syncthreads();
    s_red[tid] = v;
    __syncthreads();
    for (int w2 = kBwdThreads / 2; w2 > 0; w2 >>= 1) {
      if (tid < w2) s_red[tid] += s_red[tid + w2];
      __syncthreads();
    }
    if (tid == 0) dl_rows[int64_t(blockIdx.x) * P.q + k] = s_red[0];
  }
}

// Per-pair gradient terms from the forward sums (Phi_p, R_pq = sum_n v rb_q):
//   d Z_aq += u_p (R_pq - (z_aq - z_bq) / (2 l^2) Phi_p)  (twice for a == b)   psi_stats.hpp:297-299
// one warp per (a, q), pairs b in a fixed lane order then a shuffle tree.
template <int Q>
__global__ void __launch_bounds__(256) dir_pair_dz_kernel(PsiConst P, const double* __restrict__ u,
                                                          const double* __restrict__ sums, double* __restrict__ row) {
  const int m = P.m, mv = P.mv, lane = threadIdx.x & 31;
  const int nw = int(gridDim.x * blockDim.x) >> 5;
  auto start = [m](int r) { return int64_t(r) * m - int64_t(r) * (r - 1) / 2; };
  for (int i = int(blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m * P.q; i += nw) {
    const int a = i % m, q = i / m;
    const double il2 = 1.0 / (P.ls[q] * P.ls[q]), za = P.z64[q * m + a];
    double s = 0.0;
    for (int b = lane; b < m; b += 32) {
      const int lo = a < b ? a : b, hi = a < b ? b : a;
      const double* r = sums + (start(lo) + (hi - lo)) * (Q + 1);
      const double t = r[1 + q] - (za - P.z64[q * m + b]) * 0.5 * il2 * r[0];
      const double w = pair_weight(u, mv, lo, hi);
      s += w * (a == b ? 2.0 * t : t);
    }
    s = warp_sum_d(s);
    if (lane == 0) row[1 + P.q + a + int64_t(q) * m] = s;
  }
}

// d l_q += l sum_p u_p Phi_p (z_a - z_b)^2 / (2 l^4)   (block k < Q);  d var += 2 sum_p u_p Phi_p / var
// (block Q); fixed-order block trees (psi_stats.hpp:287, 300-303)
__global__ void __launch_bounds__(256) dir_pair_dl_kernel(PsiConst P, const double* __restrict__ u, int w1,
                                                          const double* __restrict__ sums, double* __restrict__ row) {
  __shared__ double red[256];
  const int m = P.m, mv = P.mv, k = blockIdx.x;
  const int64_t npairs = int64_t(m) * (m + 1) / 2;
  double s = 0.0;
  for (int64_t p = threadIdx.x; p < npairs; p += blockDim.x) {
    int a, b;
    pair_of(p, m, a, b);
    const double ph = sums[p * w1] * pair_weight(u, mv, a, b);
    if (k < P.q) {
      const double dz = P.z64[k * m + a] - P.z64[k * m + b], ls = P.ls[k];
      s += ph * dz * dz / (2.0 * ls * ls * ls);
    } else {
      s += ph * 2.0 / P.variance_d;
    }
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) row[k < P.q ? 1 + k : 0] = red[0];
}

// packed grads [d var, d l (Q), d Z] = d_phi n + psi1 rows (ascending) + pair row + psi2 d l rows
__global__ void dir_bwd_final_kernel(int q, int64_t count, const double* __restrict__ rows1, int nr1, int64_t rstride,
                                     const double* __restrict__ prow, const double* __restrict__ dl2, int nr2,
                                     double dvar0, int skip_pair, double* __restrict__ packed) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < count; k += int64_t(gridDim.x) * blockDim.x) {
    double s = k == 0 ? dvar0 : 0.0;
    for (int i = 0; i < nr1; ++i) s += rows1[int64_t(i) * rstride + k];
    if (!skip_pair) s += prow[k];
    if (k >= 1 && k <= q)
      for (int i = 0; i < nr2; ++i) s += dl2[int64_t(i) * q + (k - 1)];
    packed[k] = s;
  }
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
constexpr int kDirQs[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 48, 64};
int dir_q(int q) {
  for (int v : kDirQs)
    if (v >= q) return v;
  return -1;
}

struct DirFwd {
  int qi, w1;       // instantiated Q, pair-sum width (1 + qi)
  int64_t npairs, nchunks;
  int ns2, ns1, nrb; // splits of the pair sweep, of the psi1 sweep; yy/KL row blocks
  int64_t cps2, cps1;
  int64_t off_ppart, off_psum, off_p1, off_rows, doubles;
};

DirFwd dir_fwd_layout(const PsiConst& P, int num_sms) {
  DirFwd L{};
  L.qi = dir_q(P.q);
  L.w1 = L.qi + 1;
  L.npairs = int64_t(P.m) * (P.m + 1) / 2;
  L.nchunks = std::max<int64_t>(1, (P.n + kCh - 1) / kCh);
  const int64_t pb = (L.npairs + kPairThreads - 1) / kPairThreads;
  L.ns2 = int(std::min<int64_t>(L.nchunks, std::max<int64_t>(1, (4 * int64_t(num_sms) + pb - 1) / pb)));
  L.cps2 = (L.nchunks + L.ns2 - 1) / L.ns2;
  const int64_t b1 = int64_t((P.m + 31) / 32) * ((std::max(P.d, 1) + 63) / 64);
  L.ns1 = int(std::min<int64_t>(L.nchunks, std::max<int64_t>(1, (4 * int64_t(num_sms) + b1 - 1) / b1)));
  L.cps1 = (L.nchunks + L.ns1 - 1) / L.ns1;
  L.nrb = int(std::max<int64_t>(1, std::min<int64_t>((P.n + 255) / 256, 2 * int64_t(num_sms))));
  L.off_ppart = 0;
  L.off_psum = L.off_ppart + int64_t(L.ns2) * L.npairs * L.w1;
  L.off_p1 = L.off_psum + L.npairs * L.w1;
  L.off_rows = L.off_p1 + int64_t(L.ns1) * P.m * P.d;
  L.doubles = L.off_rows + 2 * int64_t(L.nrb) + 2;
  return L;
}

struct DirBwd {
  int g1, g2;
  int64_t rstride;
  int64_t off_rows1, off_prow, off_dl2, off_w, doubles;
};

DirBwd dir_bwd_layout(const PsiConst& P, int num_sms) {
  DirBwd L{};
  const int64_t ntiles = std::max<int64_t>(1, (P.n + kBwdThreads - 1) / kBwdThreads);
  L.g1 = int(std::min<int64_t>(ntiles, 4 * int64_t(num_sms)));
  L.g2 = int(std::min<int64_t>(ntiles, 8 * int64_t(num_sms)));
  L.rstride = 1 + P.q + int64_t(P.m) * P.q;
  L.off_rows1 = 0;
  L.off_prow = L.off_rows1 + int64_t(L.g1) * L.rstride;
  L.off_dl2 = L.off_prow + L.rstride;
  L.off_w = L.off_dl2 + int64_t(L.g2) * P.q + 2;
  L.doubles = L.off_w + std::max<int64_t>(P.n, 1) * P.m + 2;  // W = Y dPsi^T, N x M
  return L;
}

template <int Q>
int dir_forward_q(const PsiConst& P, double* base, double* packed, int* err_flag, int with_kl, int num_sms,
                  cudaStream_t st) {
  const DirFwd L = dir_fwd_layout(P, num_sms);
  dir_rows_kernel<<<L.nrb, 256, 0, st>>>(P, with_kl, base + L.off_rows, err_flag);
  if (P.n > 0 && P.m > 0) {
    if (P.ev_psi2[0]) record_event(P.ev_psi2[0], st);
    dir_pair_fwd_kernel<Q><<<dim3(unsigned((L.npairs + kPairThreads - 1) / kPairThreads), unsigned(L.ns2)),
                             kPairThreads, 0, st>>>(P, L.npairs, L.cps2, base + L.off_ppart);
    if (P.ev_psi2[1]) record_event(P.ev_psi2[1], st);
    if (P.d > 0)
      dir_psi1_fwd_kernel<Q><<<dim3(unsigned((P.m + 31) / 32), unsigned(L.ns1), unsigned((P.d + 63) / 64)), 256, 0,
                               st>>>(P, L.cps1 * kCh, base + L.off_p1);
  } else {
    cudaMemsetAsync(base + L.off_ppart, 0, sizeof(double) * L.ns2 * L.npairs * L.w1, st);
    cudaMemsetAsync(base + L.off_p1, 0, sizeof(double) * L.ns1 * P.m * P.d, st);
  }
  const int64_t tot = L.npairs * L.w1;
  dir_pair_reduce_kernel<<<int(std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, 4096))), 256, 0, st>>>(
      base + L.off_ppart, L.ns2, L.npairs, L.w1, base + L.off_psum, packed);
  const int64_t md = int64_t(P.m) * P.d;
  dir_fwd_final_kernel<<<int(std::max<int64_t>(1, std::min<int64_t>((md + 255) / 256, 1024))), 256, 0, st>>>(
      P, base + L.off_rows, L.nrb, base + L.off_p1, L.ns1, packed);
  g_tc_launches.fetch_add(5);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int Q>
int dir_backward_q(const PsiConst& P, const BwdConst& B, double* bbase, double* packed, int num_sms, cudaStream_t st) {
  const DirFwd F = dir_fwd_layout(P, num_sms);
  const DirBwd L = dir_bwd_layout(P, num_sms);
  const double* sums = B.fwd_rt + F.off_psum;
  double* prow = bbase + L.off_prow;
  int nr1 = 0, nr2 = 0;
  if (P.n > 0) {
    nr1 = L.g1;
    nr2 = L.g2;
    double* W = bbase + L.off_w;
    if (P.d > 0) {
      if (dla::gemm(false, true, int(P.n), P.m, P.d, 1.0, P.y, P.ld_y, B.dpsi64, P.mv, 0.0, W, P.n, st)) return 3;
    } else {
      cudaMemsetAsync(W, 0, sizeof(double) * P.n * P.m, st);
    }
    dir_psi1_bwd_kernel<Q><<<L.g1, kBwdThreads, 0, st>>>(P, B, L.rstride, bbase + L.off_rows1, W);
    if (P.ev_psi2[0]) record_event(P.ev_psi2[0], st);
    dir_pair_bwd_kernel<Q><<<L.g2, kBwdThreads, 0, st>>>(P, B, F.npairs, bbase + L.off_dl2);
    if (P.ev_psi2[1]) record_event(P.ev_psi2[1], st);
    g_tc_launches.fetch_add(2);
  }
  if (!B.skip_pair_terms) {
    dir_pair_dz_kernel<Q><<<std::max(1, (P.m * P.q + 7) / 8), 256, 0, st>>>(P, B.u64, sums, prow);
    dir_pair_dl_kernel<<<P.q + 1, 256, 0, st>>>(P, B.u64, F.w1, sums, prow);
    g_tc_launches.fetch_add(2);
  }
  dir_bwd_final_kernel<<<int(std::max<int64_t>(1, std::min<int64_t>((L.rstride + 255) / 256, 1024))), 256, 0, st>>>(
      P.q, L.rstride, bbase + L.off_rows1, nr1, L.rstride, prow, bbase + L.off_dl2, nr2, B.d_phi * double(P.n),
      B.skip_pair_terms, packed);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

#define SGPX_DIR_DISPATCH(fn, ...)      \
  switch (dir_q(P.q)) {                 \
    case 1: return fn<1>(__VA_ARGS__);  \
    case 2: return fn<2>(__VA_ARGS__);  \
    case 3: return fn<3>(__VA_ARGS__);  \
    case 4: return fn<4>(__VA_ARGS__);  \
    case 5: return fn<5>(__VA_ARGS__);  \
    case 6: return fn<6>(__VA_ARGS__);  \
    case 8: return fn<8>(__VA_ARGS__);  \
    case 10: return fn<10>(__VA_ARGS__); \
    case 12: return fn<12>(__VA_ARGS__); \
    case 16: return fn<16>(__VA_ARGS__); \
    case 20: return fn<20>(__VA_ARGS__); \
    case 24: return fn<24>(__VA_ARGS__); \
    case 32: return fn<32>(__VA_ARGS__); \
    case 48: return fn<48>(__VA_ARGS__); \
    case 64: return fn<64>(__VA_ARGS__); \
    default: return 1;                   \
  }

}  // namespace

bool direct_supported(const PsiConst& P) { return P.q >= 1 && dir_q(P.q) > 0 && P.m >= 1; }
int64_t direct_fwd_doubles(const PsiConst& P, int num_sms) { return dir_fwd_layout(P, num_sms).doubles; }
int64_t direct_bwd_doubles(const PsiConst& P, int num_sms) { return dir_bwd_layout(P, num_sms).doubles; }
double* direct_fwd_pair_sums(const PsiConst& P, double* base, int num_sms, int64_t* count) {
  const DirFwd L = dir_fwd_layout(P, num_sms);
  *count = L.npairs * L.w1;
  return base + L.off_psum;
}
int direct_forward(const PsiConst& P, double* base, double* packed, int* err_flag, int with_kl, int num_sms,
                   void* stream) {
  SGPX_DIR_DISPATCH(dir_forward_q, P, base, packed, err_flag, with_kl, num_sms, static_cast<cudaStream_t>(stream))
}
int direct_backward(const PsiConst& P, const BwdConst& B, double* bbase, double* packed, int num_sms, void* stream) {
  SGPX_DIR_DISPATCH(dir_backward_q, P, B, bbase, packed, num_sms, static_cast<cudaStream_t>(stream))
}

}  // namespace sgpx
