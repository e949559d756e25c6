// psi1_tile.cu -- psi1 statistics and gradients as tiled SIMT GEMMs (M <= 128 inducing points).
//
// Reference: psi_stats.hpp:144-219 (psi1 block of the sweep: Psi += v1^T Y, and its adjoint).
// Per chunk of 64 datapoints the CTA forms the 64 x 128 tile of weights
//
//   forward :  G_nm = v1_nm                      -> Psi_md  += sum_n G_nm y_nd        (G^T Y)
//   backward:  G_nm = v1_nm * (dPsi_m . y_n)     -> T_nk     = sum_m G_nm [1, z_m, z_m^2]   (G F)
//                                                -> R_mk    += sum_n G_nm [d1 mu, d1]_n   (G^T H)
//
// with log2 v1_nm = b1_n - (log2e / 2) sum_q d1_nq (mu_nq - z_mq)^2, d1 = 1 / (S + l^2), mu and z
// translated by the mean of Z.  Each product is a register-blocked GEMM over shared-memory tiles;
// per-inducing-point sums accumulate across chunks in fp64 (CTA-private, fixed order), and every
// CTA writes one partial row that the fixed-order row reduction sums.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <atomic>

#include "psi_common.cuh"
#include "psi_kernels.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;

namespace {
using namespace dev;

constexpr int kN = 64;     // datapoints per chunk
constexpr int kM = 128;    // inducing points per tile (the whole M)
constexpr int kGP = kM + 4;  // G row stride (floats): float4 rows, conflict-free column reads

struct Tile1Smem {  // float offsets (float4-aligned regions)
  int zq, zm, mus, d1s, b1s, ys, gs, dps, ts, hs, acc, total;
  int q4, d4;  // padded row lengths of the [m][q] / [n][d] layouts
};

// Regions: zq [Q][kM] (phase B), zm [kM][q4] (phase C, bwd), mus / d1s [Q][kN], b1 [kN],
// y (fwd: [kN][d4], bwd: [D][kN]), G [kN][kGP], bwd: dPsi^T [D][kM], T [kN][NH], H [kN][2][q4];
// fwd: Psi accumulators [D][kM] doubles.
__host__ __device__ inline Tile1Smem tile1_layout(int q, int d, bool bwd) {
  Tile1Smem L{};
  auto al4 = [](int x) { return (x + 3) / 4 * 4; };
  const int nh = 1 + 2 * q;
  L.q4 = al4(q);
  L.d4 = (d + 7) / 8 * 8;
  L.zq = 0;
  L.zm = al4(L.zq + q * kM);
  L.mus = L.zm + (bwd ? kM * L.q4 : 0);
  L.d1s = al4(L.mus + q * kN);
  L.b1s = al4(L.d1s + q * kN);
  L.ys = al4(L.b1s + kN);
  L.gs = al4(L.ys + (bwd ? d * kN : kN * L.d4));
  L.dps = al4(L.gs + kN * kGP);
  if (bwd) {
    L.ts = al4(L.dps + d * kM);
    L.hs = al4(L.ts + kN * nh);
    L.total = al4(L.hs + kN * 2 * L.q4);
    L.acc = 0;
  } else {
    L.acc = L.dps;
    L.total = L.acc + 2 * d * kM;  // d * kM doubles
  }
  return L;
}

// Phase A: per-datapoint constants (psi_stats.hpp:144-159) and the y tile [D][kN].
template <int Q>
__device__ __forceinline__ void load_chunk(const PsiConst& P, int64_t n0, float* sm, const Tile1Smem& L, int tid,
                                           int nthr, double* yy_acc, double* kl_acc, int* err_flag, bool fwd,
                                           bool fwd_layout_y) {
  const int d = P.d;
  {
    constexpr int kB = (kN * Q + 255) / 256;  // per-thread batch for 256 threads
    double mb[kB], sb[kB];
#pragma unroll
    for (int t = 0; t < kB; ++t) {
      const int i = tid + t * nthr;
      const int nl = i % kN, q = i / kN;
      const int64_t n = n0 + nl;
      const bool ok = i < kN * Q && q < P.q && n < P.n;
      mb[t] = ok ? __ldg(P.mu + q * P.ld_mu + n) : 0.0;
      sb[t] = (ok && P.expected) ? __ldg(P.s + q * P.ld_s + n) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < kB; ++t) {
      const int i = tid + t * nthr;
      if (i >= kN * Q) break;
      const int nl = i % kN, q = i / kN;
      const int64_t n = n0 + nl;
      float mu = 0.f, d1 = 0.f;
      if (q < P.q && n < P.n) {
        const double md = mb[t], sd = sb[t];
        if (fwd) {  // validation (psi_stats.hpp:119-120) + KL partial (parallel.hpp:148-149)
          if (!isfinite(md)) atomicOr(err_flag, 1);
          if (P.expected && !(sd > 0.0 && isfinite(sd))) atomicOr(err_flag, 4);
          if (P.expected) *kl_acc += 0.5 * (sd + md * md - log(sd) - 1.0);
        }
        mu = float(md - P.center[q]);
        d1 = 1.f / (float(sd) + P.l2[q]);
      }
      sm[L.mus + q * kN + nl] = mu;
      sm[L.d1s + q * kN + nl] = d1;
    }
  }
  __syncthreads();  // d1 of the chunk is staged
  for (int nl = tid; nl < kN; nl += nthr) {  // b1 = log2 var - 1/2 sum_q log2(1 + S/l^2) = log2 var + 1/2 sum log2(d1 l^2)
    const int64_t n = n0 + nl;
    float b1 = -CUDART_INF_F;
    if (n < P.n) {
      b1 = P.log2_var;
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (q < P.q) b1 += 0.5f * log2f(sm[L.d1s + q * kN + nl] * P.l2[q]);
    }
    sm[L.b1s + nl] = b1;
  }
  // y tile: batches of 8 independent loads per thread (one memory latency per batch)
  for (int i0 = tid; i0 < kN * d; i0 += 8 * nthr) {
    double yb[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = i0 + t * nthr;
      const int nl = i % kN, dd = i / kN;
      const int64_t n = n0 + nl;
      yb[t] = (i < kN * d && n < P.n) ? __ldg(P.y + dd * P.ld_y + n) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = i0 + t * nthr;
      if (i >= kN * d) break;
      const int nl = i % kN, dd = i / kN;
      const double y = yb[t];
      if (yy_acc) {
        if (fwd && !isfinite(y)) atomicOr(err_flag, 1);
        *yy_acc += y * y;
      }
      if (fwd_layout_y)
        sm[L.ys + nl * L.d4 + dd] = float(y);
      else
        sm[L.ys + dd * kN + nl] = float(y);
    }
  }
}

// Phase B: G tile [kN][kGP]; thread block of 4 datapoints x 8 inducing points, the inducing
// points split as {4 mj .. 4 mj + 3} and {64 + 4 mj .. 64 + 4 mj + 3} (16-byte spacing across the
// warp: conflict-free float4 traffic).
template <int Q, bool BWD>
__device__ __forceinline__ void build_g(const PsiConst& P, float* sm, const Tile1Smem& L, int tid) {
  const int ni = tid >> 4, mj = tid & 15;  // 16 x 16 thread grid over (64 n) x (128 m)
  const int n4 = 4 * ni, ma = 4 * mj, mb = 64 + 4 * mj;
  float c[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) c[i][j] = BWD ? 0.f : 1.f;
  if (BWD) {  // c_nm = sum_d y_nd dPsi_md
    const float* ys = sm + L.ys;
    const float* dp = sm + L.dps;
#pragma unroll 2
    for (int dd = 0; dd < P.d; ++dd) {
      const float4 y4 = *reinterpret_cast<const float4*>(ys + dd * kN + n4);
      const float4 pa = *reinterpret_cast<const float4*>(dp + dd * kM + ma);
      const float4 pb = *reinterpret_cast<const float4*>(dp + dd * kM + mb);
      const float yv[4] = {y4.x, y4.y, y4.z, y4.w}, pv[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) c[i][j] = fmaf(yv[i], pv[j], c[i][j]);
    }
  }
  float e[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) e[i][j] = 0.f;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (q >= P.q) break;
    const float4 mu4 = *reinterpret_cast<const float4*>(sm + L.mus + q * kN + n4);
    const float4 d14 = *reinterpret_cast<const float4*>(sm + L.d1s + q * kN + n4);
    const float mu[4] = {mu4.x, mu4.y, mu4.z, mu4.w}, d1[4] = {d14.x, d14.y, d14.z, d14.w};
    const float4 za = *reinterpret_cast<const float4*>(sm + L.zq + q * kM + ma);
    const float4 zb = *reinterpret_cast<const float4*>(sm + L.zq + q * kM + mb);
    const float z[8] = {za.x, za.y, za.z, za.w, zb.x, zb.y, zb.z, zb.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float df = mu[i] - z[j];
        e[i][j] = fmaf(df * df, d1[i], e[i][j]);
      }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float b1 = sm[L.b1s + n4 + i];
    float g[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int mm = j < 4 ? ma + j : mb + j - 4;
      g[j] = (mm < P.m) ? c[i][j] * ex2(fmaf(-0.5f * kLog2e, e[i][j], b1)) : 0.f;
    }
    float* gr = sm + L.gs + (n4 + i) * kGP;
    *reinterpret_cast<float4*>(gr + ma) = make_float4(g[0], g[1], g[2], g[3]);
    *reinterpret_cast<float4*>(gr + mb) = make_float4(g[4], g[5], g[6], g[7]);
  }
}

template <int Q>
__device__ __forceinline__ void load_z(const PsiConst& P, float* sm, const Tile1Smem& L, int tid, int nthr, bool zm) {
  for (int i = tid; i < Q * kM; i += nthr) {
    const int q = i / kM, mm = i % kM;
    const float z = (q < P.q && mm < P.m) ? P.zc[mm * P.qv + q] : 0.f;
    sm[L.zq + i] = z;
    if (zm) sm[L.zm + mm * L.q4 + q] = z;
  }
}

template <int Q>
__global__ void __launch_bounds__(256, 2)
    psi1_fwd_tile_kernel(PsiConst P, int64_t nchunks, double* __restrict__ part, int64_t pstride, int* err_flag,
                         int with_kl) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int d = P.d;
  const Tile1Smem L = tile1_layout(Q, d, false);
  double* psi_acc = reinterpret_cast<double*>(sm + L.acc);  // [d][kM]
  load_z<Q>(P, sm, L, tid, nthr, false);
  for (int i = tid; i < d * kM; i += nthr) psi_acc[i] = 0.0;
  double yy_acc = 0.0, kl_acc = 0.0;
  // Psi phase: thread tile of 4 inducing points x 8 outputs dims (32 m-groups x 8 d-groups per
  // 64-wide pass over d); G float4 along m, y float4 along d (broadcast within the d-group)
  const int mg = tid & 31, dgp = tid >> 5;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    __syncthreads();
    load_chunk<Q>(P, chunk * kN, sm, L, tid, nthr, &yy_acc, &kl_acc, err_flag, with_kl != 0, true);
    __syncthreads();
    build_g<Q, false>(P, sm, L, tid);
    __syncthreads();
    // Psi_md += sum_n G_nm y_nd   (fp32 over the chunk, fp64 across chunks)
    for (int db = 8 * dgp; db < d; db += 64) {
      float acc[4][8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[i][k] = 0.f;
#pragma unroll 4
      for (int nl = 0; nl < kN; ++nl) {
        const float4 g4 = *reinterpret_cast<const float4*>(sm + L.gs + nl * kGP + 4 * mg);
        const float* yr = sm + L.ys + nl * L.d4 + db;
        const float4 ya = *reinterpret_cast<const float4*>(yr);
        const float4 yb = *reinterpret_cast<const float4*>(yr + 4);
        const float gv[4] = {g4.x, g4.y, g4.z, g4.w}, yv[8] = {ya.x, ya.y, ya.z, ya.w, yb.x, yb.y, yb.z, yb.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[i][k] = fmaf(gv[i], yv[k], acc[i][k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (db + k < d)
#pragma unroll
          for (int i = 0; i < 4; ++i) psi_acc[(db + k) * kM + 4 * mg + i] += double(acc[i][k]);
    }
  }
  __syncthreads();
  double* const cta_part = part + int64_t(blockIdx.x) * pstride;
  double* const psi_part = cta_part + 2 + int64_t(P.m) * (P.m + 1) / 2;
  for (int i = tid; i < d * kM; i += nthr) {
    const int m_ = i % kM, dd = i / kM;
    if (m_ < P.m) psi_part[m_ + int64_t(dd) * P.m] = psi_acc[i];
  }
  __shared__ double red[2][8];
  yy_acc = warp_sum_d(yy_acc);
  kl_acc = warp_sum_d(kl_acc);
  if (lane == 0) {
    red[0][warp] = yy_acc;
    red[1][warp] = kl_acc;
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, k = 0.0;
    for (int i = 0; i < nthr / 32; ++i) {
      s += red[0][i];
      k += red[1][i];
    }
    cta_part[0] = s;
    if (with_kl) cta_part[1] = k;
  }
}

template <int Q>
__global__ void __launch_bounds__(256, 2)
    psi1_bwd_tile_kernel(PsiConst P, BwdConst B, int64_t nchunks, double* __restrict__ part, int64_t pstride) {
  extern __shared__ __align__(16) float sm[];
  constexpr int NH = 1 + 2 * Q;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int d = P.d, m = P.m;
  const Tile1Smem L = tile1_layout(Q, d, true);
  const int q4 = L.q4;
  float* dps = sm + L.dps;  // dPsi^T [d][kM]
  float* ts = sm + L.ts;    // T [kN][NH]
  float* hs = sm + L.hs;    // H [kN][2][q4]: d1 mu, d1
  load_z<Q>(P, sm, L, tid, nthr, true);
  for (int i = tid; i < d * kM; i += nthr) {
    const int mm = i % kM, dd = i / kM;
    dps[i] = mm < m ? B.dpsi[dd * P.mv + mm] : 0.f;
  }
  // per-inducing-point sums R_mk (k < 2Q) in fp64: thread (m, half of k)
  const int mm = tid & (kM - 1), kg = tid >> 7;
  double racc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) racc[q] = 0.0;
  double dl_acc[Q], dv_acc = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q) dl_acc[q] = 0.0;
  const double inv_var = 1.0 / P.variance_d;
  // per-datapoint sums: four lanes per datapoint, inducing points interleaved mod 4
  const int tn = tid >> 2, tq = tid & 3;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int64_t n0 = chunk * kN;
    __syncthreads();
    load_chunk<Q>(P, n0, sm, L, tid, nthr, nullptr, nullptr, nullptr, false, false);
    __syncthreads();
    build_g<Q, true>(P, sm, L, tid);
    for (int i = tid; i < Q * kN; i += nthr) {  // H = [d1 mu, d1]
      const int nl = i % kN, q = i / kN;
      const float d1 = sm[L.d1s + q * kN + nl];
      hs[nl * 2 * q4 + q] = d1 * sm[L.mus + q * kN + nl];
      hs[nl * 2 * q4 + q4 + q] = d1;
    }
    __syncthreads();
    // T_nk = sum_m G_nm [1, z_m, z_m^2]
    {
      float t0 = 0.f, t1[Q], t2[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) t1[q] = t2[q] = 0.f;
      const float* gr = sm + L.gs + tn * kGP;
      for (int m_ = tq; m_ < m; m_ += 4) {
        const float g = gr[m_];
        const float* zr = sm + L.zm + m_ * q4;
        t0 += g;
#pragma unroll
        for (int q = 0; q < Q; q += 4) {
          const float4 z4 = *reinterpret_cast<const float4*>(zr + q);
          const float zz[4] = {z4.x, z4.y, z4.z, z4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (q + u < Q) {
              const float gz = g * zz[u];
              t1[q + u] += gz;
              t2[q + u] = fmaf(gz, zz[u], t2[q + u]);
            }
        }
      }
      // combine the four lanes of this datapoint (fixed order)
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        t0 += __shfl_xor_sync(0xffffffffu, t0, o);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          t1[q] += __shfl_xor_sync(0xffffffffu, t1[q], o);
          t2[q] += __shfl_xor_sync(0xffffffffu, t2[q], o);
        }
      }
      if (tq == 0) {
        ts[tn * NH] = t0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          ts[tn * NH + 1 + q] = t1[q];
          ts[tn * NH + 1 + Q + q] = t2[q];
        }
      }
    }
    // R_mk += sum_n G_nm H_nk
    {
      float r[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) r[q] = 0.f;
#pragma unroll 2
      for (int nl = 0; nl < kN; ++nl) {
        const float g = sm[L.gs + nl * kGP + mm];
        const float* hr = hs + nl * 2 * q4 + kg * q4;
#pragma unroll
        for (int q = 0; q < Q; q += 4) {
          const float4 h4 = *reinterpret_cast<const float4*>(hr + q);
          const float hh[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (q + u < Q) r[q + u] = fmaf(g, hh[u], r[q + u]);
        }
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) racc[q] += double(r[q]);
    }
    __syncthreads();
    // per-datapoint epilogue (psi_stats.hpp:200-219): d mu, d S (+ KL), d l, d var
    for (int i = tid; i < kN * Q; i += nthr) {
      const int nl = i / Q, q = i - nl * Q;
      const int64_t n = n0 + nl;
      if (q >= P.q || n >= P.n) continue;
      const double p0 = ts[nl * NH], p1 = ts[nl * NH + 1 + q], p2 = ts[nl * NH + 1 + Q + q];
      const double mu = sm[L.mus + q * kN + nl], dd1 = sm[L.d1s + q * kN + nl];
      const double s = P.expected ? P.s[q * P.ld_s + n] : 0.0, l = P.ls[q];
      const double q1 = mu * mu * p0 - 2.0 * mu * p1 + p2;
      double dlv = s * dd1 * p0 / l + l * dd1 * dd1 * q1;
#pragma unroll
      for (int qq = 0; qq < Q; ++qq)
        if (qq == q) dl_acc[qq] += dlv;
      if (q == 0) dv_acc += p0 * inv_var;
      if (B.write_local) {
        double dmu = -dd1 * (mu * p0 - p1);
        double ds = -0.5 * dd1 * p0 + 0.5 * dd1 * dd1 * q1;
        if (B.add_kl) {  // KL(q || N(0, I)) enters the bound with a minus sign (parallel.hpp:163-166)
          dmu -= P.mu[q * P.ld_mu + n];
          ds -= 0.5 * (1.0 - 1.0 / s);
        }
        B.d_mu[q * B.ld_g + n] = dmu;
        if (P.expected) B.d_s[q * B.ld_g + n] = ds;
      }
    }
  }
  // d z_mq = R_mq - z_mq R_m(Q+q)   (psi_stats.hpp:214), exchanged through shared memory
  __syncthreads();
  double* rsh = reinterpret_cast<double*>(sm + L.gs);  // [2Q][kM] doubles (G tile and beyond are free now)
#pragma unroll
  for (int q = 0; q < Q; ++q) rsh[(kg * Q + q) * kM + mm] = racc[q];
  __syncthreads();
  double* const row = part + int64_t(blockIdx.x) * pstride;
  for (int i = tid; i < m * P.q; i += nthr) {
    const int m_ = i % m, q = i / m;
    const double z = sm[L.zq + q * kM + m_];
    row[1 + P.q + m_ + int64_t(q) * m] = rsh[q * kM + m_] - z * rsh[(Q + q) * kM + m_];
  }
  // d l, d var: fixed-order block reduction
  __syncthreads();
  double* red = reinterpret_cast<double*>(sm + L.gs);
  for (int k = 0; k <= P.q; ++k) {
    double v = k < P.q ? 0.0 : dv_acc;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (q == k && k < P.q) v = dl_acc[q];  // k == P.q is d var (a padded template Q has q == P.q)
    red[tid] = v;
    __syncthreads();
    for (int w = nthr / 2; w > 0; w >>= 1) {
      if (tid < w) red[tid] += red[tid + w];
      __syncthreads();
    }
    if (tid == 0) row[k < P.q ? 1 + k : 0] = red[0];
    __syncthreads();
  }
}

template <int Q>
int launch_tile_fwd(const PsiConst& P, double* part, int64_t pstride, int rows, int* err_flag, int with_kl,
                    cudaStream_t st) {
  const Tile1Smem L = tile1_layout(Q, P.d, false);
  const size_t smem = sizeof(float) * size_t(L.total);
  auto kern = psi1_fwd_tile_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  const int64_t nchunks = (P.n + kN - 1) / kN;
  if (rows > 0) {
    kern<<<rows, 256, smem, st>>>(P, nchunks, part, pstride, err_flag, with_kl);
    g_tc_launches.fetch_add(1);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int Q>
int launch_tile_bwd(const PsiConst& P, const BwdConst& B, double* part, int64_t pstride, int rows, cudaStream_t st) {
  const Tile1Smem L = tile1_layout(Q, P.d, true);
  const size_t smem = sizeof(float) * size_t(L.total);
  auto kern = psi1_bwd_tile_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 3;
  const int64_t nchunks = (P.n + kN - 1) / kN;
  if (rows > 0) {
    kern<<<rows, 256, smem, st>>>(P, B, nchunks, part, pstride);
    g_tc_launches.fetch_add(1);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

#define SGPX_T1_DISPATCH(FN, ...)        \
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

}  // namespace

bool psi1_tile_supported(const PsiConst& P, bool bwd) {
  if (P.m < 1 || P.m > kM || P.q < 1) return false;
  const int q = instantiated_q(P.q);
  const Tile1Smem L = tile1_layout(q, P.d, bwd);
  if (bwd && size_t(2) * q * kM * sizeof(double) > sizeof(float) * size_t(L.total - L.gs)) return false;
  return sizeof(float) * size_t(L.total) <= 227 * 1024;
}
int psi1_tile_rows(const PsiConst& P, int num_sms) {
  const int64_t nchunks = (P.n + kN - 1) / kN;
  return int(std::min<int64_t>(nchunks, int64_t(num_sms) * 2));
}
int psi1_tile_forward(const PsiConst& P, double* part, int64_t pstride, int rows, int* err_flag, int with_kl,
                      void* stream) {
  SGPX_T1_DISPATCH(launch_tile_fwd, P, part, pstride, rows, err_flag, with_kl, static_cast<cudaStream_t>(stream))
}
int psi1_tile_backward(const PsiConst& P, const BwdConst& B, double* part, int64_t pstride, int rows, void* stream) {
  SGPX_T1_DISPATCH(launch_tile_bwd, P, B, part, pstride, rows, static_cast<cudaStream_t>(stream))
}

}  // namespace sgpx
