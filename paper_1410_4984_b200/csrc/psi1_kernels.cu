// psi1_kernels.cu -- the psi1 half of the statistics / gradient passes as standalone kernels
// (used with the tensor-core psi2 kernels so those carry no psi1 prologue).
//
// Reference: psi_stats.hpp:172-219 (psi1 blocks: Psi_m += sum_n v1_nm y_n; backward with
// w_n = <y_n, dPsi_m>) and Worker::pass KL terms (parallel.hpp:148-149, 163-166).
//
//   psi1_fwd_kernel : CTA-cooperative chunks of 32 datapoints; Psi = Psi1^T Y as 4x4 register
//                     tiles; writes yy and Psi into the fp64 CTA partial row (forward layout).
//   psi1_bwd_kernel : one warp per chunk of 32 datapoints (no block barriers in the loop);
//                     G1_nm = v1_nm <y_n, dPsi_m>; writes d_mu / d_s = psi1 part (+ KL) as the
//                     first writer, and per-warp partial rows [d_variance, d_l, d_z].
#include <cuda_runtime.h>

#include <algorithm>
#include <math_constants.h>

#include <atomic>

#include "psi_common.cuh"
#include "psi_kernels.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;

namespace {
using namespace dev;

template <int Q>
__global__ void __launch_bounds__(256, 2)
    psi1_fwd_kernel(PsiConst P, int64_t nchunks, double* __restrict__ part, int64_t pstride, int* err_flag,
                    int with_kl, int n_sacc) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, nthr = blockDim.x;
  const int m = P.m, mv = P.mv, qv = P.qv, d = P.d, dv = P.dv;
  float* Zc = sm;
  float* V1s = Zc + mv * qv;   // [32][mv]
  float* Ys = V1s + 32 * mv;   // [32][dv]
  double* red = reinterpret_cast<double*>(Ys + 32 * dv);  // [2][32]
  for (int i = tid; i < mv * qv; i += nthr) Zc[i] = P.zc[i];
  __syncthreads();
  const int64_t npairs = int64_t(m) * (m + 1) / 2;
  double* const cta_part = part + int64_t(blockIdx.x) * pstride;
  double* const psi_part = cta_part + 2 + npairs;
  const int DT = dv >> 2;
  const int ntiles1 = (mv >> 2) * DT;
  double yy_acc = 0.0, kl_acc = 0.0;
  // Psi tiles t < n_sacc accumulate in fp64 in shared memory across all chunks of this CTA (each
  // tile has one owning thread; layout [16][n_sacc] so a warp's accesses are conflict-free); the
  // CTA is the single writer of its partial row.  Tiles beyond n_sacc fall back to RED.ADD.F64.
  double* sacc = red + 64;
  for (int i = tid; i < 16 * n_sacc; i += nthr) sacc[i] = 0.0;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int64_t n = chunk * 32 + lane;
    const bool valid = n < P.n;
    const int64_t nn = valid ? n : 0;
    // all raw loads first (one memory latency per chunk)
    double md[Q], sd[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int qq = q < P.q ? q : 0;
      md[q] = __ldg(P.mu + qq * P.ld_mu + nn);
      sd[q] = P.expected ? __ldg(P.s + qq * P.ld_s + nn) : 0.0;
    }
    // per-lane psi1 constants (psi_stats.hpp:144-159): centred mu, 1/(S+l^2), log2 c1
    float mu[Q], d1[Q], b1 = P.log2_var;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      mu[q] = 0.f;
      d1[q] = 0.f;
      if (q < P.q && valid) {
        const float sv = float(sd[q]);
        if (with_kl && (q % nw) == warp) {  // validation (psi_stats.hpp:119-120) + KL (parallel.hpp:148-149)
          if (!isfinite(md[q])) atomicOr(err_flag, 1);
          if (P.expected && !(sd[q] > 0.0 && isfinite(sd[q]))) atomicOr(err_flag, 4);
          if (P.expected) kl_acc += 0.5 * (sd[q] + md[q] * md[q] - log(sd[q]) - 1.0);
        }
        mu[q] = float(md[q] - P.center[q]);
        d1[q] = 1.f / (sv + P.l2[q]);
        b1 += -0.5f * log2f(1.f + sv * P.il2[q]);
      }
    }
    if (!valid) b1 = -CUDART_INF_F;
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
#pragma unroll 4
    for (int dd = warp; dd < dv; dd += nw) {
      const double y0 = (dd < d && valid) ? __ldg(P.y + dd * P.ld_y + n) : 0.0;
      if (!isfinite(y0)) atomicOr(err_flag, 1);
      yy_acc += y0 * y0;
      Ys[lane * dv + dd] = float(y0);
    }
    __syncthreads();
    for (int t = tid; t < ntiles1; t += nthr) {
      const int mt = t / DT, dt = t - mt * DT;
      float acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[r][j] = 0.f;
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const float4 vv = *reinterpret_cast<const float4*>(V1s + k * mv + 4 * mt);
        const float4 yv = *reinterpret_cast<const float4*>(Ys + k * dv + 4 * dt);
        const float va[4] = {vv.x, vv.y, vv.z, vv.w}, ya[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[r][j] = fmaf(va[r], ya[j], acc[r][j]);
      }
      if (t < n_sacc) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j) sacc[(4 * r + j) * n_sacc + t] += double(acc[r][j]);
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int mm = 4 * mt + r, dd = 4 * dt + j;
            if (mm < m && dd < d) atomicAdd(psi_part + mm + int64_t(dd) * m, double(acc[r][j]));
          }
      }
    }
    __syncthreads();
  }
  for (int t = tid; t < n_sacc; t += nthr) {
    const int mt = t / DT, dt = t - mt * DT;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int mm = 4 * mt + r, dd = 4 * dt + j;
        if (mm < m && dd < d) psi_part[mm + int64_t(dd) * m] = sacc[(4 * r + j) * n_sacc + t];
      }
  }
  yy_acc = warp_sum_d(yy_acc);
  kl_acc = warp_sum_d(kl_acc);
  if (lane == 0) {
    red[warp] = yy_acc;
    red[32 + warp] = kl_acc;
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, k = 0.0;
    for (int i = 0; i < nw; ++i) {
      s += red[i];
      k += red[32 + i];
    }
    cta_part[0] = s;
    if (with_kl) cta_part[1] = k;
  }
}

template <int Q>
__global__ void __launch_bounds__(256, 2)
    psi1_bwd_kernel(PsiConst P, BwdConst B, int64_t nchunks, double* __restrict__ part, int64_t pstride) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, nthr = blockDim.x;
  const int m = P.m, mv = P.mv, qv = P.qv, d = P.d;
  float* Zc = sm;
  float* Dps = Zc + mv * qv;     // dPsi^T [d][mv]
  float* Ys = Dps + d * mv + warp * (d * 32);  // this warp's y tile [d][32]
  for (int i = tid; i < mv * qv; i += nthr) Zc[i] = P.zc[i];
  for (int i = tid; i < d * mv; i += nthr) Dps[i] = B.dpsi[i];
  __syncthreads();
  const int64_t wrow = int64_t(blockIdx.x) * nw + warp;  // per-warp partial row (single writer)
  double* const wpart = part + wrow * pstride;
  double* const dz_part = wpart + 1 + P.q;
  double dl_acc[Q], dv_acc = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q) dl_acc[q] = 0.0;
  const double inv_var = 1.0 / P.variance_d;
  constexpr int QR = Q <= 8 ? 8 : (Q <= 16 ? 16 : 32), SH = QR == 8 ? 2 : (QR == 16 ? 1 : 0);

  for (int64_t chunk = int64_t(blockIdx.x) * nw + warp; chunk < nchunks; chunk += int64_t(gridDim.x) * nw) {
    const int64_t n = chunk * 32 + lane;
    const bool valid = n < P.n;
    float mu[Q], d1[Q], sv[Q], b1 = P.log2_var;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      mu[q] = 0.f;
      d1[q] = 0.f;
      sv[q] = 0.f;
      if (q < P.q && valid) {
        const double md = P.mu[q * P.ld_mu + n];
        sv[q] = P.expected ? float(P.s[q * P.ld_s + n]) : 0.f;
        mu[q] = float(md - P.center[q]);
        d1[q] = 1.f / (sv[q] + P.l2[q]);
        b1 += -0.5f * log2f(1.f + sv[q] * P.il2[q]);
      }
    }
    if (!valid) b1 = -CUDART_INF_F;
#pragma unroll 4
    for (int dd = 0; dd < d; ++dd) Ys[dd * 32 + lane] = valid ? float(P.y[dd * P.ld_y + n]) : 0.f;
    __syncwarp();
    float p0 = 0.f, p1[Q], p2[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) p1[q] = p2[q] = 0.f;
    for (int mt = 0; mt < (mv >> 2); ++mt) {
      float w4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 5
      for (int dd = 0; dd < d; ++dd) {
        const float yv = Ys[dd * 32 + lane];
        const float4 dp = *reinterpret_cast<const float4*>(Dps + dd * mv + 4 * mt);
        w4[0] = fmaf(yv, dp.x, w4[0]);
        w4[1] = fmaf(yv, dp.y, w4[1]);
        w4[2] = fmaf(yv, dp.z, w4[2]);
        w4[3] = fmaf(yv, dp.w, w4[3]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int mm = 4 * mt + i;
        float z[Q];
        load_z<Q>(Zc + mm * qv, z);
        float e = 0.f;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const float df = mu[q] - z[q];
          e = fmaf(df * df, d1[q], e);
        }
        const float g = (mm < m) ? w4[i] * ex2(fmaf(-0.5f * kLog2e, e, b1)) : 0.f;
        p0 += g;
        float vr[QR];
#pragma unroll
        for (int q = 0; q < QR; ++q) vr[q] = 0.f;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          p1[q] = fmaf(g, z[q], p1[q]);
          p2[q] = fmaf(g * z[q], z[q], p2[q]);
          vr[q] = g * d1[q] * (mu[q] - z[q]);  // d z_mq contribution (psi_stats.hpp:214)
        }
        const float tot = reduce_scatter<QR>(vr, lane);
        const int qi = lane >> SH;
        if (mm < m && qi < P.q && (lane & ((1 << SH) - 1)) == 0) atomicAdd(dz_part + mm + int64_t(qi) * m, double(tot));
      }
    }
    if (valid) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (q >= P.q) break;
        const double muq = mu[q], s = sv[q], l = P.ls[q];
        const double dd1 = d1[q];
        const double q1 = muq * muq * p0 - 2.0 * muq * p1[q] + p2[q];
        dl_acc[q] += s * dd1 * p0 / l + l * dd1 * dd1 * q1;
        if (B.write_local) {
          double dmu = -dd1 * (muq * p0 - p1[q]);
          double ds = -0.5 * dd1 * p0 + 0.5 * dd1 * dd1 * q1;
          if (B.add_kl) {  // KL(q || N(0, I)) enters the bound with a minus sign (parallel.hpp:163-166)
            const double mo = P.mu[q * P.ld_mu + n], so = P.s[q * P.ld_s + n];
            dmu -= mo;
            ds -= 0.5 * (1.0 - 1.0 / so);
          }
          B.d_mu[q * B.ld_g + n] = dmu;
          B.d_s[q * B.ld_g + n] = ds;
        }
      }
      dv_acc += p0 * inv_var;
    }
    __syncwarp();
  }
  // fixed-order warp reductions into this warp's row
  dv_acc = warp_sum_d(dv_acc);
#pragma unroll
  for (int q = 0; q < Q; ++q) dl_acc[q] = warp_sum_d(dl_acc[q]);
  if (lane == 0) {
    wpart[0] = dv_acc;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (q < P.q) wpart[1 + q] = dl_acc[q];
  }
}

template <int Q>
int launch_psi1_fwd_q(const PsiConst& P, double* part_rows, int64_t pstride, int rows, int* err_flag,
                      cudaStream_t st, int with_kl) {
  const int64_t nchunks = (P.n + 31) / 32;
  const size_t base = sizeof(float) * (size_t(P.mv) * P.qv + 32 * size_t(P.mv) + 32 * size_t(P.dv)) +
                      64 * sizeof(double);
  // shared fp64 Psi accumulators: as many tiles as fit next to two resident CTAs per SM
  const int ntiles1 = (P.mv / 4) * (P.dv / 4);
  const size_t budget = 110 * 1024;
  const int n_sacc = base >= budget ? 0 : int(std::min<size_t>(ntiles1, (budget - base) / (16 * sizeof(double))));
  const size_t smem = base + size_t(n_sacc) * 16 * sizeof(double);
  auto kern = psi1_fwd_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  if (rows > 0) {
    kern<<<rows, 256, smem, st>>>(P, nchunks, part_rows, pstride, err_flag, with_kl, n_sacc);
    g_tc_launches.fetch_add(1);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int Q>
int launch_psi1_bwd_q(const PsiConst& P, const BwdConst& B, double* part_rows, int64_t pstride, int ctas,
                      cudaStream_t st) {
  const int64_t nchunks = (P.n + 31) / 32;
  const size_t smem = sizeof(float) * (size_t(P.mv) * P.qv + size_t(P.d) * P.mv + 8 * 32 * size_t(P.d));
  auto kern = psi1_bwd_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  if (ctas > 0) {
    kern<<<ctas, 256, smem, st>>>(P, B, nchunks, part_rows, pstride);
    g_tc_launches.fetch_add(1);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

// Partial rows the psi1 kernels write (callers size their partial buffers with these).
int psi1_fwd_rows(const PsiConst& P, int num_sms) {
  if (psi1_tc_supported(P, false)) return psi1_tc_rows(P, num_sms, false);
  if (psi1_tile_supported(P, false)) return psi1_tile_rows(P, num_sms);
  const int64_t nchunks = (P.n + 31) / 32;
  return int(std::min<int64_t>(nchunks, int64_t(num_sms) * 2));
}
int psi1_bwd_ctas(const PsiConst& P, int num_sms) {
  const int64_t nwchunks = (P.n + 31) / 32;
  return int(std::max<int64_t>(1, std::min<int64_t>((nwchunks + 7) / 8, int64_t(num_sms) * 3)));
}
int psi1_bwd_rows(const PsiConst& P, int num_sms) {
  if (psi1_tc_supported(P, true)) return psi1_tc_rows(P, num_sms, true);
  if (psi1_tile_supported(P, true)) return std::max(1, psi1_tile_rows(P, num_sms));
  return 8 * psi1_bwd_ctas(P, num_sms);
}

#define SGPX_P1_DISPATCH(FN, ...)        \
  switch (instantiated_q(P.q)) {         \
    case 1: return FN<1>(__VA_ARGS__);   \
    case 2: return FN<2>(__VA_ARGS__);   \
    case 3: return FN<3>(__VA_ARGS__);   \
    case 4: return FN<4>(__VA_ARGS__);   \
    case 5: return FN<5>(__VA_ARGS__);   \
    case 6: return FN<6>(__VA_ARGS__);   \
    case 8: return FN<8>(__VA_ARGS__);   \
    case 10: return FN<10>(__VA_ARGS__); \
    case 12: return FN<12>(__VA_ARGS__); \
    case 16: return FN<16>(__VA_ARGS__); \
    case 20: return FN<20>(__VA_ARGS__); \
    case 24: return FN<24>(__VA_ARGS__); \
    case 32: return FN<32>(__VA_ARGS__); \
    default: return 1;                   \
  }

int psi1_forward(const PsiConst& P, double* part_rows, int64_t pstride, int rows, int* err_flag, void* stream,
                 int with_kl) {
  if (psi1_tc_supported(P, false)) return psi1_tc_forward(P, part_rows, pstride, rows, err_flag, with_kl, stream);
  if (psi1_tile_supported(P, false)) return psi1_tile_forward(P, part_rows, pstride, rows, err_flag, with_kl, stream);
  SGPX_P1_DISPATCH(launch_psi1_fwd_q, P, part_rows, pstride, rows, err_flag, static_cast<cudaStream_t>(stream), with_kl)
}

int psi1_backward(const PsiConst& P, const BwdConst& B, double* part_rows, int64_t pstride, int rows,
                  void* stream) {
  if (psi1_tc_supported(P, true)) return psi1_tc_backward(P, B, part_rows, pstride, rows, stream);
  if (psi1_tile_supported(P, true)) return psi1_tile_backward(P, B, part_rows, pstride, rows, stream);
  const int ctas = rows / 8;
  SGPX_P1_DISPATCH(launch_psi1_bwd_q, P, B, part_rows, pstride, ctas, static_cast<cudaStream_t>(stream))
}

}  // namespace sgpx
