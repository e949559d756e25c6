// dcoord.cu -- the coordinator of Engine::evaluate on the device.
//
// Reference: factor_gram (kernels.hpp:177-197), bound_core (bound.hpp:84-119), adjoints_from_core
// (bound.hpp:196-226), kern_grads(Z, Z, dKmm) (kernels.hpp:124-164) and the gradient assembly of
// Engine::evaluate (parallel.hpp:378-421).  The same fp64 algebra as coordinator.cpp, restated as a
// sequence of stream-ordered kernels, so that one evaluation (forward psi pass -> allreduce #1 ->
// coordinator -> backward psi pass -> allreduce #2 -> assembly) never waits on the host and can be
// replayed as one CUDA graph.  Numeric breakdowns (no Cholesky at the largest jitter, a non-finite
// bound) and contract violations of the reduced statistics set a status word that the host reads
// with the results and turns into the reference's exceptions.
//
//   per broadcast   Kmm (no jitter), factor_gram escalation -> L_k, log|Kmm|, W_k = L_k^-1,
//                   Kmm^-1 = W_k^T W_k
//   after AR #1     A = Kmm + jitter + beta Phi, factor_spd escalation -> L_a, log|A|, A^-1, G = A^-1 Psi,
//                   G G^T, the bound terms, d Phi / d Psi as the fp32 operands of the backward kernels,
//                   then (off the backward's critical path) Kmm^-1 Phi Kmm^-1, d Kmm, Phi G, d beta
//   after AR #2     kern_grads(Z, Z, d Kmm) + the jitter term, final gradient vector
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>

#include "dcoord.cuh"
#include "dla.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;

namespace {

constexpr double kLog2Pi = 1.8378770664093454835606594728112;

// Kmm without jitter: var exp(-1/2 sum_q (z_aq - z_bq)^2 / l_q^2) (kern_gram, kernels.hpp:83-112).
__global__ void gram_kernel(const double* __restrict__ z, int m, int q, const double* __restrict__ ls, double var,
                            double* __restrict__ kmm) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= int64_t(m) * m) return;
  const int a = int(e % m), b = int(e / m);
  double d2 = 0.0;
  for (int j = 0; j < q; ++j) {
    const double d = (z[a + int64_t(j) * m] - z[b + int64_t(j) * m]) / ls[j];
    d2 += d * d;
  }
  kmm[e] = a == b ? var : var * exp(-0.5 * d2);
}

// A = Kmm + jitter I + beta Phi (Phi mirrored from the packed upper triangle).
__global__ void build_a_kernel(const double* __restrict__ kmm, const double* __restrict__ packed, int m, double beta,
                               double var, const double* __restrict__ sc, double* __restrict__ a) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= int64_t(m) * m) return;
  const int i = int(e % m), j = int(e / m);
  const int lo = min(i, j), hi = max(i, j);
  const double phi = packed[4 + int64_t(lo) * m - int64_t(lo) * (lo - 1) / 2 + (hi - lo)];
  const double jit = i == j ? sc[kScJitterFactor] * var : 0.0;
  a[e] = kmm[e] + jit + beta * phi;
}

// Phi (mirrored) into a dense M x M matrix.
__global__ void unpack_phi_kernel(const double* __restrict__ packed, int m, double* __restrict__ phi) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= int64_t(m) * m) return;
  const int i = int(e % m), j = int(e / m);
  const int lo = min(i, j), hi = max(i, j);
  phi[e] = packed[4 + int64_t(lo) * m - int64_t(lo) * (lo - 1) / 2 + (hi - lo)];
}

__device__ double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double s = red[0];
  __syncthreads();
  return s;
}

__device__ __forceinline__ double dev_warp_sum(double v) {  // fixed butterfly order
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Bound terms (bound.hpp:108-116) and the scalar adjoint d_phi; contract checks of the reduced
// statistics (bound.hpp:84-92).  One CTA, fixed-order trees.
__global__ void __launch_bounds__(1024) bound_kernel(DcArgs A) {
  __shared__ double red[1024];
  const int m = A.m, d = A.d;
  const double* packed = A.packed;
  const double* psi = packed + 4 + int64_t(m) * (m + 1) / 2;
  double pg = 0.0, kp = 0.0, ap = 0.0;
  for (int64_t e = threadIdx.x; e < int64_t(m) * d; e += blockDim.x) pg += psi[e] * A.g[e];
  for (int64_t e = threadIdx.x; e < int64_t(m) * m; e += blockDim.x) {
    kp += A.kinv[e] * A.phi[e];
    ap += A.ainv[e] * A.phi[e];
  }
  pg = block_sum(pg, red);
  kp = block_sum(kp, red);
  ap = block_sum(ap, red);
  if (threadIdx.x == 0) {
    double* sc = A.sc;
    int st = int(sc[kScStatus]);
    const double beta = A.beta, nd = double(A.n), dd = double(d);
    const double phi0 = packed[0], yy = packed[1], nc = packed[2], kl = packed[3];
    if (!(nc == nd)) st |= kStBadCount;
    if (!(phi0 >= 0.0 && yy >= 0.0)) st |= kStBadStats;
    const double logdet_k = sc[kScLogDetK], logdet_a = sc[kScLogDetA];
    double* bd = sc + kScBound;
    bd[1] = dd * (0.5 * nd * log(beta) + 0.5 * logdet_k - 0.5 * nd * kLog2Pi - 0.5 * logdet_a);
    bd[2] = -0.5 * beta * yy;
    bd[3] = 0.5 * beta * beta * pg;
    bd[4] = -0.5 * beta * dd * phi0;
    bd[5] = 0.5 * beta * dd * kp;
    bd[6] = A.latent ? -kl : 0.0;
    bd[0] = bd[1] + bd[2] + bd[3] + bd[4] + bd[5] + bd[6];
    if (!isfinite(bd[0])) st |= kStNonFinite;
    sc[kScPg] = pg;
    sc[kScKp] = kp;
    sc[kScAp] = ap;
    sc[kScDPhi] = -0.5 * beta * dd;
    sc[kScStatus] = double(st);
  }
}

// d Phi = -1/2 beta D A^-1 - 1/2 beta^3 G G^T + 1/2 beta D Kmm^-1 (bound.hpp:203-210), mirrored into
// the fp32 [mv][mv] operand of the backward kernels, and d Psi^T = beta^2 G^T as fp32 [d][mv].
__global__ void adjoint_kernel(DcArgs A, float* __restrict__ u, float* __restrict__ dpsi, double* __restrict__ u64,
                               double* __restrict__ dpsi64) {
  const int m = A.m, mv = A.mv, d = A.d;
  const double beta = A.beta, dd = double(d);
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e < int64_t(mv) * mv) {
    const int i = int(e % mv), j = int(e / mv);
    double v = 0.0;
    if (i < m && j < m) {
      const int64_t k = i + int64_t(j) * m;
      v = -0.5 * beta * dd * A.ainv[k] - 0.5 * beta * beta * beta * A.ggt[k] + 0.5 * beta * dd * A.kinv[k];
    }
    u[e] = float(v);  // symmetric: A^-1, G G^T, Kmm^-1 are exactly symmetric products
    u64[e] = v;
  }
  if (e < int64_t(max(d, 1)) * mv) {
    const int a = int(e % mv), dc = int(e / mv);
    const double v = (a < m && dc < d) ? beta * beta * A.g[a + int64_t(dc) * m] : 0.0;
    dpsi[e] = float(v);
    dpsi64[e] = v;
  }
}

// d Kmm (bound.hpp:211-216) = 1/2 D Kmm^-1 - 1/2 D A^-1 - 1/2 beta^2 G G^T - 1/2 beta D sym(Kmm^-1 Phi Kmm^-1)
__global__ void dkmm_kernel(DcArgs A) {
  const int m = A.m;
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= int64_t(m) * m) return;
  const int i = int(e % m), j = int(e / m);
  const double beta = A.beta, dd = double(A.d);
  const double kpk = 0.5 * (A.kpk[e] + A.kpk[j + int64_t(i) * m]);
  A.dkmm[e] = 0.5 * dd * A.kinv[e] - 0.5 * dd * A.ainv[e] - 0.5 * beta * beta * A.ggt[e] - 0.5 * beta * dd * kpk;
}

// d beta (bound.hpp:217-223) and kern_grads(Z, Z, d Kmm) with the gradient assembly of
// parallel.hpp:414-421 (d_z + d_x, d var + jitter_factor tr(d Kmm), d l).  One CTA.
// W = d Kmm o K (K without jitter), the first step of kern_grads(Z, Z, U) (kernels.hpp:124-164)
__global__ void w_kernel(DcArgs A) {
  const int64_t mm = int64_t(A.m) * A.m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < mm; e += int64_t(gridDim.x) * blockDim.x)
    A.w[e] = A.dkmm[e] * A.kmm[e];
}
// row sums of W, thread per row, ascending b (coalesced across rows)
__global__ void rowsum_kernel(DcArgs A) {
  const int m = A.m;
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  double s = 0.0;
  for (int b = 0; b < m; ++b) s += A.w[a + int64_t(b) * m];
  A.rs[a] = s;
}

// the tail of the gradient assembly, after W, rs and W Z (one CTA, fixed-order block sums)
__global__ void __launch_bounds__(1024) finish_kernel(DcArgs A, const double* __restrict__ pgrads) {
  __shared__ double red[1024];
  const int m = A.m, q = A.q, d = A.d;
  const double beta = A.beta, nd = double(A.n), dd = double(d);
  double* sc = A.sc;
  // tr(G^T Phi G)
  double tg = 0.0;
  for (int64_t e = threadIdx.x; e < int64_t(m) * d; e += blockDim.x) tg += A.g[e] * A.phig[e];
  tg = block_sum(tg, red);
  // sum W = sum of the row sums, trace of d Kmm
  double tot = 0.0, tr = 0.0;
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    tot += A.rs[a];
    tr += A.dkmm[a + int64_t(a) * m];
  }
  tot = block_sum(tot, red);
  tr = block_sum(tr, red);
  double* res = A.result;  // [d var, d l (Q), d Z (M Q), d beta]
  for (int64_t e = threadIdx.x; e < int64_t(m) * q; e += blockDim.x) {
    const int a = int(e % m), j = int(e / m);
    const double il2 = 1.0 / (A.ls[j] * A.ls[j]);
    res[1 + q + e] = pgrads[1 + q + e] + 2.0 * (A.wz[e] - A.rs[a] * A.z[e]) * il2;
  }
  // sum_ab W_ab (z_a - z_b)^2 = 2 (sum_a rs_a z_a^2 - z^T W z) per dimension (a warp per q, fixed tree)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < q; j += blockDim.x >> 5) {
    double s2 = 0.0, cross = 0.0;
    for (int a = lane; a < m; a += 32) {
      const double za = A.z[a + int64_t(j) * m];
      s2 += A.rs[a] * za * za;
      cross += za * A.wz[a + int64_t(j) * m];
    }
    s2 = dev_warp_sum(s2);
    cross = dev_warp_sum(cross);
    if (lane == 0) res[1 + j] = pgrads[1 + j] + 2.0 * (s2 - cross) / (A.ls[j] * A.ls[j] * A.ls[j]);
  }
  if (threadIdx.x == 0) {
    res[0] = pgrads[0] + tot / A.var + sc[kScJitterFactor] * tr;
    const double yy = A.packed[1], phi0 = A.packed[0];
    res[1 + q + int64_t(m) * q] = 0.5 * dd * nd / beta - 0.5 * dd * sc[kScAp] - 0.5 * yy + beta * sc[kScPg] -
                                  0.5 * beta * beta * tg - 0.5 * dd * phi0 + 0.5 * dd * sc[kScKp];
  }
}

// ---------------------------------------------------------------------------------------------
// Small-M path (M <= kSmallM): each coordinator step is ONE CTA working in shared memory —
// right-looking Cholesky (1 barrier per column), L^-1 a warp per column, the products by 4 x 4
// register tiles.
// ---------------------------------------------------------------------------------------------
constexpr int kSmallM = 112;  // 2 M^2 doubles of shared memory (<= 200 KB)
__device__ long long g_dc_prof[16];  // SGPX debug: clock64 phase stamps of bound_small_kernel
#define DC_STAMP(i) \
  if (threadIdx.x == 0) g_dc_prof[i] = clock64()

// Right-looking lower Cholesky of the shared m x m matrix L (lower triangle valid) in place, one
// barrier per column: step j subtracts a_ij a_cj / a_jj from the trailing lower triangle with the
// still-unscaled column j (a 32 x 32 thread grid over (row, column) offsets, no index division),
// the columns are scaled by l_jj = sqrt(a_jj) once at the end.  dg: m doubles of scratch (l_jj).
__device__ bool chol_right_smem(double* L, int m, double* dg) {
  const int tr = threadIdx.x & 31, tc = threadIdx.x >> 5, nc = blockDim.x >> 5;
  for (int j = 0; j < m; ++j) {
    const double d = L[j + j * m];
    if (!(d > 0.0)) {
      __syncthreads();
      return false;
    }
    if (threadIdx.x == 0) dg[j] = sqrt(d);
    const double inv = 1.0 / d;
    const int R = m - j - 1;
    const double* cj = L + j * m + j + 1;  // a_(j+1..m-1), j
    for (int r = tr; r < R; r += 32) {
      const double lr = cj[r] * inv;
      for (int c = tc; c <= r; c += nc) L[(j + 1 + r) + (j + 1 + c) * m] -= lr * cj[c];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e % m, j = e / m;
    if (i > j) L[e] /= dg[j];
    else if (i == j) L[e] = dg[j];
  }
  __syncthreads();
  return true;
}

// W = L^-1 (lower): a warp per column j, the column in registers (lane l owns rows l + 32 t),
// column-oriented substitution in the host's order (x_k /= L_kk, then x_i -= L_ik x_k).  Stored
// row-major (S[k m + j] = W_kj), zeros above the diagonal.  m <= 128.
__device__ void trinv_warp_smem(const double* L, double* S, int m) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < m; j += nw) {
    double x[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) x[t] = (lane + 32 * t == j) ? 1.0 : 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (32 * t + 31 < j || 32 * t >= m) continue;
      for (int l = 0; l < 32; ++l) {
        const int k = 32 * t + l;
        if (k < j) continue;
        if (k >= m) break;
        const double xk = __shfl_sync(0xffffffffu, x[t], l) / L[k + k * m];
        if (lane == l) x[t] = xk;
#pragma unroll
        for (int u = t; u < 4; ++u) {
          const int i = lane + 32 * u;
          if (i > k && i < m) x[u] -= L[i + k * m] * xk;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = lane + 32 * t;
      if (i < m) S[i * m + j] = x[t];
    }
  }
}

// C = A B with a(i, p), b(p, j) element accessors: 4 x 4 register tiles, one per thread, p ascending
// (each element a single fma chain in a fixed order); c(i, j, value) stores.
// C = A B on the fp64 tensor cores (mma.sync m8n8k4 .f64: the same 64 FMA/clk/SM as DFMA, one
// instruction per 256 FMAs instead of 32 -- the small-M coordinator is instruction-bound, not
// FMA-bound).  Strided operands A(i, p) = a[i ai + p ap], B(p, j) = b[p bp + j bj] (shared or global
// memory); a warp per 16 x 16 tile of C (2 x 2 mma tiles), k ascending in steps of 4 (fixed order:
// deterministic); c(i, j, value) stores.  Fragments (PTX m8n8k4 f64): A row = lane / 4, col = lane % 4;
// B row = lane % 4, col = lane / 4; C row = lane / 4, cols 2 (lane % 4) + {0, 1}.
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
template <class FC>
__device__ void mma_gemm(int m, int n, int k, const double* __restrict__ a, int ai, int ap, const double* __restrict__ b,
                         int bp, int bj, FC c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int tm = (m + 15) / 16, tn = (n + 15) / 16;
  for (int tile = warp; tile < tm * tn; tile += nw) {
    const int i0 = (tile % tm) * 16, j0 = (tile / tm) * 16;
    double acc[2][2][2] = {};
    const int ia0 = i0 + g, ia1 = i0 + 8 + g, jb0 = j0 + g, jb1 = j0 + 8 + g;
    const bool ra0 = ia0 < m, ra1 = ia1 < m, cb0 = jb0 < n, cb1 = jb1 < n;
    const double* pa0 = a + int64_t(ra0 ? ia0 : 0) * ai;
    const double* pa1 = a + int64_t(ra1 ? ia1 : 0) * ai;
    const double* pb0 = b + int64_t(cb0 ? jb0 : 0) * bj;
    const double* pb1 = b + int64_t(cb1 ? jb1 : 0) * bj;
    auto fetch = [&](int p0, double& a0, double& a1, double& b0, double& b1) {
      const int pp = p0 + t;
      const bool kp = pp < k;
      const int64_t oa = int64_t(kp ? pp : 0) * ap, ob = int64_t(kp ? pp : 0) * bp;
      a0 = (kp && ra0) ? pa0[oa] : 0.0;
      a1 = (kp && ra1) ? pa1[oa] : 0.0;
      b0 = (kp && cb0) ? pb0[ob] : 0.0;
      b1 = (kp && cb1) ? pb1[ob] : 0.0;
    };
    double a0, a1, b0, b1;
    fetch(0, a0, a1, b0, b1);
    for (int p0 = 0; p0 < k; p0 += 4) {  // the next k-step's operands load under this step's MMAs
      double na0 = 0.0, na1 = 0.0, nb0 = 0.0, nb1 = 0.0;
      if (p0 + 4 < k) fetch(p0 + 4, na0, na1, nb0, nb1);
      dmma(acc[0][0], a0, b0);
      dmma(acc[0][1], a0, b1);
      dmma(acc[1][0], a1, b0);
      dmma(acc[1][1], a1, b1);
      a0 = na0, a1 = na1, b0 = nb0, b1 = nb1;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = i0 + 8 * r + g, j = j0 + 8 * q + 2 * t + h;
          if (i < m && j < n) c(i, j, acc[r][q][h]);
        }
  }
}

// X = W^T W from the row-major S (W lower triangular: the terms below the diagonal range are exact
// zeros; both triangles from the same products in the same order) -> out (and out2 if given)
__device__ void wtw_smem(const double* S, int m, double* out, double* out2 = nullptr) {
  mma_gemm(
      m, m, m, S, 1, m, S, m, 1,
      [&](int i, int j, double v) {
        out[i + j * m] = v;
        if (out2) out2[i + j * m] = v;
      });
}

__device__ double block_sum_s(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double s = red[0];
  __syncthreads();
  return s;
}

// Factor the shared matrix rebuilt by `fill(shift)` with the escalation schedule of `mode` (see
// chol_kernel); returns the factor used through *fac, log det through *logdet.
template <class Fill>
__device__ bool factor_smem(double* L, int m, int mode, double f0, double var, double scale, Fill fill, double* red,
                            int* s_flag, double* fac, double* logdet) {
  double f = mode == 0 ? f0 : 0.0;
  bool ok = false;
  for (int attempt = 0; attempt < 32; ++attempt) {
    fill(mode == 0 ? f * var : f * scale);
    __syncthreads();
    ok = chol_right_smem(L, m, red);
    __syncthreads();
    if (threadIdx.x == 0) {
      g_dc_prof[10 + mode] = attempt + 1;
      g_dc_prof[12 + mode] = ok;
    }
    if (ok) break;
    if (mode == 0) {
      if (f >= 1e-2) break;
      f = f == 0.0 ? 1e-6 : f * 10.0;
    } else {
      f = f == 0.0 ? 1e-10 : f * 10.0;
      if (!(f <= 1e-2)) break;
    }
  }
  double s = 0.0;
  if (ok)
    for (int i = threadIdx.x; i < m; i += blockDim.x) s += log(L[i + i * m]);
  s = block_sum_s(s, red);
  *fac = f;
  *logdet = 2.0 * s;
  return ok;
}

__global__ void __launch_bounds__(1024) prefactor_small_kernel(DcArgs A) {
  extern __shared__ double sm[];
  __shared__ double red[1024];
  __shared__ int s_flag;
  const int m = A.m, q = A.q;
  double* L = sm;
  double* W = sm + m * m;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {  // Kmm without jitter (kern_gram)
    const int a = e % m, b = e / m;
    double d2 = 0.0;
    for (int j = 0; j < q; ++j) {
      const double d = (A.z[a + int64_t(j) * m] - A.z[b + int64_t(j) * m]) / A.ls[j];
      d2 += d * d;
    }
    A.kmm[e] = a == b ? A.var : A.var * exp(-0.5 * d2);
  }
  __syncthreads();
  double fac = 0.0, ld = 0.0;
  const bool ok = factor_smem(
      L, m, 0, A.jitter_factor, A.var, 0.0,
      [&](double shift) {
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) L[e] = A.kmm[e] + (e % m == e / m ? shift : 0.0);
      },
      red, &s_flag, &fac, &ld);
  if (ok) {
    trinv_warp_smem(L, W, m);
    __syncthreads();
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) A.wk[e] = W[(e % m) * m + e / m];  // L_k^-1 (prediction)
    wtw_smem(W, m, A.kinv);
  }
  if (threadIdx.x == 0) {
    A.sc[kScLogDetK] = ld;
    A.sc[kScJitterFactor] = fac;
    A.sc[kScStatusK] = ok ? 0.0 : double(kStGramFailed);
  }
}

__global__ void __launch_bounds__(1024) bound_small_kernel(DcArgs A, float* __restrict__ u, float* __restrict__ dpsi,
                                                           double* __restrict__ u64, double* __restrict__ dpsi64) {
  extern __shared__ double sm[];
  __shared__ double red[1024];
  __shared__ int s_flag;
  const int m = A.m, d = A.d, mv = A.mv;
  double* L = sm;
  double* W = sm + m * m;
  const double* packed = A.packed;
  const double* psi = packed + 4 + int64_t(m) * (m + 1) / 2;
  const double beta = A.beta, jit = A.sc[kScJitterFactor] * A.var;
  DC_STAMP(0);
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e % m, j = e / m, lo = min(i, j), hi = max(i, j);
    A.phi[e] = packed[4 + int64_t(lo) * m - int64_t(lo) * (lo - 1) / 2 + (hi - lo)];
  }
  __syncthreads();
  double mx = 0.0;  // factor_spd's scale: max |a_ii|
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    mx = fmax(mx, fabs(A.kmm[i + i * m] + jit + beta * A.phi[i + i * m]));
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  const double scale = red[0];
  __syncthreads();
  double fac = 0.0, ld = 0.0;
  const bool ok = factor_smem(
      L, m, 1, 0.0, 0.0, scale,
      [&](double shift) {
        for (int e = threadIdx.x; e < m * m; e += blockDim.x)
          L[e] = A.kmm[e] + beta * A.phi[e] + (e % m == e / m ? jit + shift : 0.0);
      },
      red, &s_flag, &fac, &ld);
  DC_STAMP(1);
  if (ok) {
    trinv_warp_smem(L, W, m);
    __syncthreads();
    DC_STAMP(2);
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) A.wa[e] = W[(e % m) * m + e / m];  // L_a^-1 (prediction)
    __syncthreads();
    wtw_smem(W, m, L, A.ainv);  // A^-1 into shared memory (over L) and global
  }
  __syncthreads();
  DC_STAMP(3);
  // G = A^-1 Psi (M x D): A^-1 from shared memory, Psi through the read-only path; G into shared memory
  // over W when it fits (M D <= M^2), else global only
  double* gs = d <= m ? W : nullptr;
  mma_gemm(
      m, d, m, L, 1, m, psi, 1, m,
      [&](int i, int j, double v) {
        A.g[i + int64_t(j) * m] = v;
        if (gs) gs[i + j * m] = v;
      });
  __syncthreads();
  const double* gg = gs ? gs : A.g;
  mma_gemm(
      m, m, d, gg, 1, m, gg, m, 1, [&](int i, int j, double v) { A.ggt[i + j * m] = v; });
  __syncthreads();
  DC_STAMP(4);
  // reductions and the bound terms (bound.hpp:108-116)
  double pg = 0.0, kp = 0.0, ap = 0.0;
  for (int64_t e = threadIdx.x; e < int64_t(m) * d; e += blockDim.x) pg += __ldg(psi + e) * gg[e];
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const double ph = A.phi[e];
    kp += __ldg(A.kinv + e) * ph;
    ap += L[e] * ph;
  }
  pg = block_sum_s(pg, red);
  kp = block_sum_s(kp, red);
  ap = block_sum_s(ap, red);
  if (threadIdx.x == 0) {
    double* sc = A.sc;
    int st = int(sc[kScStatusK]) | (ok ? 0 : kStAFailed);
    const double nd = double(A.n), dd = double(d);
    const double phi0 = packed[0], yy = packed[1], nc = packed[2], kl = packed[3];
    if (!(nc == nd)) st |= kStBadCount;
    if (!(phi0 >= 0.0 && yy >= 0.0)) st |= kStBadStats;
    double* bd = sc + kScBound;
    bd[1] = dd * (0.5 * nd * log(beta) + 0.5 * sc[kScLogDetK] - 0.5 * nd * kLog2Pi - 0.5 * ld);
    bd[2] = -0.5 * beta * yy;
    bd[3] = 0.5 * beta * beta * pg;
    bd[4] = -0.5 * beta * dd * phi0;
    bd[5] = 0.5 * beta * dd * kp;
    bd[6] = A.latent ? -kl : 0.0;
    bd[0] = bd[1] + bd[2] + bd[3] + bd[4] + bd[5] + bd[6];
    if (!isfinite(bd[0])) st |= kStNonFinite;
    sc[kScLogDetA] = ld;
    sc[kScShiftA] = fac;
    sc[kScPg] = pg;
    sc[kScKp] = kp;
    sc[kScAp] = ap;
    sc[kScDPhi] = -0.5 * beta * dd;
    sc[kScStatus] = double(st);
  }
  __syncthreads();
  DC_STAMP(5);
  // the backward's operands (bound.hpp:203-210)
  const double dd = double(d);
  for (int e = threadIdx.x; e < mv * mv; e += blockDim.x) {
    const int i = e % mv, j = e / mv;
    double v = 0.0;
    if (i < m && j < m) {
      const int k = i + j * m;
      v = -0.5 * beta * dd * L[k] - 0.5 * beta * beta * beta * A.ggt[k] + 0.5 * beta * dd * __ldg(A.kinv + k);
    }
    u[e] = float(v);
    u64[e] = v;
  }
  for (int64_t e = threadIdx.x; e < int64_t(max(d, 1)) * mv; e += blockDim.x) {
    const int a = int(e % mv), c = int(e / mv);
    const double v = (a < m && c < d) ? beta * beta * gg[a + int64_t(c) * m] : 0.0;
    dpsi[e] = float(v);
    dpsi64[e] = v;
  }
}

// ---------------------------------------------------------------------------------------------
// Split small-M coordinator: the backward's psi1 kernel needs only d Psi = beta^2 G, so
//   K1 (bound_g_small_kernel, on the evaluation's stream): A = Kmm + jitter + beta Phi, factor_spd
//       escalation, log|A|, G = A^-1 Psi, d Psi, <Psi, G>;
//   K2 (bound_u_small_kernel, on a side stream, concurrent with the psi1 backward): L^-1, A^-1, G G^T,
//       the bound terms and d Phi (= U, the psi2 backward's operand); then deferred_small_kernel.
// K1 is a blocked right-looking Cholesky with 32-column panels: one warp factors the diagonal block,
// the 32 warps invert it (a warp per column), and the panel below (TRSM, as A_21 D^-T), the trailing
// update (SYRK) and both triangular solves for G are fp64 tensor-core GEMMs -- a block-wide barrier
// per phase instead of one per column, and ~8x fewer instructions than per-element updates.
// ---------------------------------------------------------------------------------------------
constexpr int kG1Rhs = 64;      // right-hand-side columns per solve chunk
constexpr int kG1Threads = 512;  // 128 registers: the diagonal block lives in one warp's registers
size_t g_small_smem(int m) {  // L (m x m), D^-1 blocks (4 x 32 x 32), X (m x kG1Rhs), Tmp (max(m, 64) x 32)
  return sizeof(double) * (size_t(m) * m + 4 * 32 * 32 + size_t(m) * kG1Rhs + size_t(std::max(m, 64)) * 32);
}

__global__ void __launch_bounds__(kG1Threads) bound_g_small_kernel(DcArgs A, float* __restrict__ dpsi,
                                                             double* __restrict__ dpsi64) {
  extern __shared__ double sm[];
  __shared__ double red[1024];
  __shared__ double invd[128], diag[128];
  __shared__ int s_fail;
  const int m = A.m, d = A.d, mv = A.mv;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nt = blockDim.x;
  const int nb = (m + 31) / 32;
  double* L = sm;                  // A, factored in place (lower triangle)
  double* Wd = L + m * m;          // inverse of diagonal block b at Wd + 1024 b (32 x 32, column-major, lower)
  double* X = Wd + 4 * 1024;       // m x kG1Rhs right-hand sides (leading dimension m)
  double* Tmp = X + m * kG1Rhs;    // m x 32 scratch
  const double* packed = A.packed;
  const double* psi = packed + 4 + int64_t(m) * (m + 1) / 2;
  const double beta = A.beta, jit = A.sc[kScJitterFactor] * A.var;
  auto phi_at = [&](int i, int j) {
    const int lo = min(i, j), hi = max(i, j);
    return packed[4 + int64_t(lo) * m - int64_t(lo) * (lo - 1) / 2 + (hi - lo)];
  };
  DC_STAMP(0);
  double f = 0.0, scale = 0.0;  // factor_spd escalation (bound.hpp:52-62): shift f * max |a_ii|
  bool ok = false;
  for (int attempt = 0; attempt < 32; ++attempt) {
    if (attempt == 1) {  // the matrix's own scale, needed from the first retry on
      double mx = 0.0;
      for (int i = threadIdx.x; i < m; i += nt) mx = fmax(mx, fabs(A.kmm[i + i * m] + jit + beta * phi_at(i, i)));
      red[threadIdx.x] = mx;
      __syncthreads();
      for (int w = nt / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
      }
      scale = red[0];
      __syncthreads();
    }
    const double shift = f * scale;
    for (int e = threadIdx.x; e < m * m; e += nt) {
      const int i = e % m, j = e / m;
      const double ph = phi_at(i, j);
      if (attempt == 0) A.phi[e] = ph;  // dense Phi (K2, deferred)
      L[e] = A.kmm[e] + beta * ph + (i == j ? jit + shift : 0.0);
    }
    for (int e = threadIdx.x; e < 4 * 1024; e += nt) Wd[e] = 0.0;
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    DC_STAMP(1);
    for (int b = 0; b < nb; ++b) {
      const int j0 = 32 * b, jb = min(32, m - j0), mr = m - j0 - jb;
      double* Lp = L + j0 + j0 * m;  // the diagonal block
      if (warp == 0) {  // (1) factor the diagonal block: right-looking inside one warp (lane = row, in place)
        const int r = lane;
        for (int k = 0; k < jb; ++k) {
          const double dkk = Lp[k + k * m];
          const bool bad = !(dkk > 0.0);
          const double inv = bad ? 1.0 : rsqrt(dkk), lkk = bad ? 1.0 : dkk * inv;
          double lrk = 0.0;
          if (r > k && r < jb) {
            lrk = Lp[r + k * m] * inv;
            Lp[r + k * m] = lrk;
          }
          if (r == k) {
            Lp[k + k * m] = lkk;
            invd[j0 + k] = inv;
            diag[j0 + k] = lkk;
            if (bad) s_fail = 1;
          }
          __syncwarp();
          // row r, columns k + 1 .. r: every candidate column's loads first (predicated, compile-time
          // register indices in halves of 16), then the FMAs and stores (tools/microbench/diag_factor.cu)
          const bool rowact = r > k && r < jb;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (16 * h + 15 <= k) continue;  // warp-uniform
            double av[16], lv[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const int c = 16 * h + u;
              const bool act = rowact && c > k && c <= r;
              av[u] = act ? Lp[r + c * m] : 0.0;
              lv[u] = act ? Lp[c + k * m] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const int c = 16 * h + u;
              if (rowact && c > k && c <= r) Lp[r + c * m] = fma(-lrk, lv[u], av[u]);
            }
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (b == 0) DC_STAMP(5);
      if (s_fail) break;
      // (2) D^-1: a warp per column c, the block's 32 rows one per lane
      double* W = Wd + 1024 * b;
      for (int c = warp; c < jb; c += nt / 32) {
        double x = lane == c ? 1.0 : 0.0;
        for (int k = c; k < jb; ++k) {
          const double xk = __shfl_sync(0xffffffffu, x, k) * invd[j0 + k];
          if (lane == k) x = xk;
          if (lane > k && lane < jb) x -= Lp[lane + k * m] * xk;
        }
        W[lane + 32 * c] = (lane >= c && lane < jb) ? x : 0.0;
      }
      __syncthreads();
      if (b == 0) DC_STAMP(6);
      if (mr > 0) {
        // (3) panel below: L_21 = A_21 D^-T  (Tmp, mr x jb)
        double* A21 = L + (j0 + jb) + j0 * m;
        mma_gemm(mr, jb, jb, A21, 1, m, W, 32, 1, [&](int i, int j, double v) { Tmp[i + j * mr] = v; });
        __syncthreads();
        for (int e = threadIdx.x; e < mr * jb; e += nt) A21[(e % mr) + (e / mr) * m] = Tmp[e];
        __syncthreads();
        if (b == 0) DC_STAMP(7);
        // (4) trailing update A_22 -= L_21 L_21^T (lower triangle)
        double* A22 = L + (j0 + jb) + (j0 + jb) * m;
        mma_gemm(mr, mr, jb, A21, 1, m, A21, m, 1, [&](int i, int j, double v) {
          if (i >= j) A22[i + j * m] -= v;
        });
        __syncthreads();
        if (b == 0) DC_STAMP(8);
      }
    }
    __syncthreads();
    ok = !s_fail;
    __syncthreads();
    if (ok) break;
    f = f == 0.0 ? 1e-10 : f * 10.0;
    if (!(f <= 1e-2)) break;
  }
  DC_STAMP(2);
  // log |A| (fixed-order tree over log l_ii)
  double s = 0.0;
  if (ok)
    for (int i = threadIdx.x; i < m; i += nt) s += log(diag[i]);
  s = block_sum_s(s, red);
  for (int e = threadIdx.x; e < m * m; e += nt) {  // the factor (zero upper triangle): prediction
    const int i = e % m, j = e / m;
    A.la[e] = i >= j ? L[e] : 0.0;
    if (i < j) L[e] = 0.0;  // (A's upper triangle is still there)
  }
  __syncthreads();
  if (ok) {
    // W = L^-1 in place of L, block row by block row: W_ii = D_i^-1, W_i,<i = -D_i^-1 (L_i,<i W_<i,<i)
    for (int bi = 0; bi < nb; ++bi) {
      const int i0 = 32 * bi, ib = min(32, m - i0);
      if (bi > 0) {
        mma_gemm(ib, i0, i0, L + i0, 1, m, L, 1, m, [&](int r, int c, double v) { Tmp[r + c * 32] = v; });
        __syncthreads();
        mma_gemm(ib, i0, ib, Wd + 1024 * bi, 1, 32, Tmp, 1, 32,
                 [&](int r, int c, double v) { L[(i0 + r) + c * m] = -v; });
      }
      for (int e = threadIdx.x; e < ib * ib; e += nt) {
        const int r = e % ib, c = e / ib;
        L[(i0 + r) + (i0 + c) * m] = r >= c ? Wd[1024 * bi + r + 32 * c] : 0.0;
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < m * m; e += nt) {  // L_a^-1 (K2's A^-1, prediction), zero upper triangle
      const int i = e % m, j = e / m;
      A.wa[e] = i >= j ? L[e] : 0.0;
      L[e] = i >= j ? L[e] : 0.0;
    }
    __syncthreads();
  }
  // G = W^T (W Psi) in chunks of 32 columns, Psi staged in shared memory
  for (int c0 = 0; c0 < d; c0 += 32) {
    const int nc = min(32, d - c0);
    if (ok) {
      for (int e = threadIdx.x; e < m * nc; e += nt) X[e] = psi[int64_t(c0) * m + e];
      __syncthreads();
      mma_gemm(m, nc, m, L, 1, m, X, 1, m, [&](int i, int j, double v) { Tmp[i + j * m] = v; });
      __syncthreads();
      mma_gemm(m, nc, m, L, m, 1, Tmp, 1, m, [&](int i, int j, double v) { A.g[int64_t(c0 + j) * m + i] = v; });
    } else {
      for (int e = threadIdx.x; e < m * nc; e += nt) A.g[int64_t(c0) * m + e] = psi[int64_t(c0) * m + e];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < mv * nc; e += nt) {
      const int i = e % mv, j = c0 + e / mv;
      const double v = i < m ? beta * beta * A.g[i + int64_t(j) * m] : 0.0;
      dpsi[int64_t(j) * mv + i] = float(v);
      dpsi64[int64_t(j) * mv + i] = v;
    }
    __syncthreads();
  }
  DC_STAMP(3);
  double pg = 0.0;  // <Psi, G> (bound.hpp:108-116), fixed-order tree
  for (int64_t e = threadIdx.x; e < int64_t(m) * d; e += nt) pg += psi[e] * A.g[e];
  pg = block_sum_s(pg, red);
  if (threadIdx.x == 0) {
    A.sc[kScLogDetA] = 2.0 * s;
    A.sc[kScShiftA] = f;
    A.sc[kScPg] = pg;
    A.sc[kScStatus] = double(int(A.sc[kScStatusK]) | (ok ? 0 : kStAFailed));
  }
  DC_STAMP(4);
}

// K2: L^-1, A^-1 = W^T W, G G^T, the bound terms and status, d Phi (U) as the psi2 backward's operands.
__global__ void __launch_bounds__(1024) bound_u_small_kernel(DcArgs A, float* __restrict__ u,
                                                             double* __restrict__ u64) {
  extern __shared__ double sm[];
  __shared__ double red[1024];
  const int m = A.m, d = A.d, mv = A.mv;
  double* L = sm;
  double* W = sm + m * m;
  const double* packed = A.packed;
  const double beta = A.beta;
  const bool ok = !(int(A.sc[kScStatus]) & kStAFailed);
  if (ok) {
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) W[(e % m) * m + e / m] = A.wa[e];  // K1's L^-1, row-major
    __syncthreads();
    wtw_smem(W, m, L, A.ainv);  // A^-1 into shared memory (over L) and global
  }
  __syncthreads();
  // G G^T with G (K1's output) staged over W when it fits
  double* gs = d <= m ? W : nullptr;
  if (gs)
    for (int e = threadIdx.x; e < m * d; e += blockDim.x) gs[e] = A.g[e];
  __syncthreads();
  const double* gg = gs ? gs : A.g;
  mma_gemm(
      m, m, d, gg, 1, m, gg, m, 1, [&](int i, int j, double v) { A.ggt[i + j * m] = v; });
  __syncthreads();
  double kp = 0.0, ap = 0.0;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const double ph = A.phi[e];
    kp += A.kinv[e] * ph;
    ap += L[e] * ph;
  }
  kp = block_sum_s(kp, red);
  ap = block_sum_s(ap, red);
  if (threadIdx.x == 0) {
    double* sc = A.sc;
    int st = int(sc[kScStatus]);
    const double nd = double(A.n), dd = double(d);
    const double phi0 = packed[0], yy = packed[1], nc = packed[2], kl = packed[3];
    if (!(nc == nd)) st |= kStBadCount;
    if (!(phi0 >= 0.0 && yy >= 0.0)) st |= kStBadStats;
    double* bd = sc + kScBound;
    const double pg = sc[kScPg];
    bd[1] = dd * (0.5 * nd * log(beta) + 0.5 * sc[kScLogDetK] - 0.5 * nd * kLog2Pi - 0.5 * sc[kScLogDetA]);
    bd[2] = -0.5 * beta * yy;
    bd[3] = 0.5 * beta * beta * pg;
    bd[4] = -0.5 * beta * dd * phi0;
    bd[5] = 0.5 * beta * dd * kp;
    bd[6] = A.latent ? -kl : 0.0;
    bd[0] = bd[1] + bd[2] + bd[3] + bd[4] + bd[5] + bd[6];
    if (!isfinite(bd[0])) st |= kStNonFinite;
    sc[kScKp] = kp;
    sc[kScAp] = ap;
    sc[kScDPhi] = -0.5 * beta * dd;
    sc[kScStatus] = double(st);
  }
  __syncthreads();
  const double dd = double(d);
  for (int e = threadIdx.x; e < mv * mv; e += blockDim.x) {  // bound.hpp:203-210
    const int i = e % mv, j = e / mv;
    double v = 0.0;
    if (i < m && j < m) {
      const int k = i + j * m;
      v = -0.5 * beta * dd * L[k] - 0.5 * beta * beta * beta * A.ggt[k] + 0.5 * beta * dd * A.kinv[k];
    }
    u[e] = float(v);
    u64[e] = v;
  }
}

__global__ void dc_prof_kernel(long long* out) {
  if (threadIdx.x < 16) out[threadIdx.x] = g_dc_prof[threadIdx.x];
}

// d Kmm (with Kmm^-1 Phi Kmm^-1), Phi G, d beta, kern_grads(Z, Z, d Kmm), the assembly: one CTA.
// part 1: Kmm^-1 Phi Kmm^-1 (needs only the statistics: runs concurrently with K1 in the split
// coordinator); part 2: the rest (after K2); part 0: both.
__global__ void __launch_bounds__(1024) deferred_small_kernel(DcArgs A, int part) {
  extern __shared__ double sm[];
  const int m = A.m, d = A.d;
  double* K = sm;          // Kmm^-1
  double* T = sm + m * m;  // Phi, then Kmm^-1 Phi
  if (part != 2) {
    const double* packed = A.packed;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = e % m, j = e / m, lo = min(i, j), hi = max(i, j);
      K[e] = A.kinv[e];
      T[e] = packed[4 + int64_t(lo) * m - int64_t(lo) * (lo - 1) / 2 + (hi - lo)];
    }
    __syncthreads();
    mma_gemm(  // tmp = Kmm^-1 Phi
        m, m, m, K, 1, m, T, 1, m, [&](int i, int j, double v) { A.tmp[i + j * m] = v; });
    __syncthreads();
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) T[e] = A.tmp[e];
    __syncthreads();
    mma_gemm(  // kpk = tmp Kmm^-1
        m, m, m, T, 1, m, K, 1, m, [&](int i, int j, double v) { A.kpk[i + j * m] = v; });
    if (part == 1) return;
    __syncthreads();
  }
  if (d <= m) {  // Phi G with both operands staged in shared memory (Phi dense from K1)
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) T[e] = A.phi[e];
    for (int e = threadIdx.x; e < m * d; e += blockDim.x) K[e] = A.g[e];
    __syncthreads();
    mma_gemm(m, d, m, T, 1, m, K, 1, m, [&](int i, int j, double v) { A.phig[i + int64_t(j) * m] = v; });
  } else {
    mma_gemm(m, d, m, A.phi, 1, m, A.g, 1, m, [&](int i, int j, double v) { A.phig[i + int64_t(j) * m] = v; });
  }
  __syncthreads();
  const double beta = A.beta, dd = double(d);
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e % m, j = e / m;
    const double kpk = 0.5 * (A.kpk[e] + A.kpk[j + i * m]);
    const double dk =
        0.5 * dd * A.kinv[e] - 0.5 * dd * A.ainv[e] - 0.5 * beta * beta * A.ggt[e] - 0.5 * beta * dd * kpk;
    A.dkmm[e] = dk;
    K[e] = dk * A.kmm[e];  // W = d Kmm o K (kern_grads(Z, Z, d Kmm), kernels.hpp:124-164)
  }
  __syncthreads();
  // everything of the assembly (parallel.hpp:414-421) that does not depend on the backward's
  // statistics, into A.result; finish_add_kernel adds the psi gradients
  __shared__ double red[1024];
  const int q = A.q, mq = m * q;
  double* rs = A.rs;
  for (int a = threadIdx.x; a < m; a += blockDim.x) {  // row sums of W, ascending b
    double r = 0.0;
    for (int b = 0; b < m; ++b) r += K[a + b * m];
    rs[a] = r;
  }
  mma_gemm(m, q, m, K, 1, m, A.z, 1, m, [&](int i, int j, double v) { A.wz[i + j * m] = v; });  // W Z
  __syncthreads();
  double tg = 0.0;  // tr(G^T Phi G)
  for (int64_t e = threadIdx.x; e < int64_t(m) * d; e += blockDim.x) tg += A.g[e] * A.phig[e];
  tg = block_sum(tg, red);
  double tot = 0.0, tr = 0.0;  // sum W, trace of d Kmm
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    tot += rs[a];
    tr += A.dkmm[a + a * m];
  }
  tot = block_sum(tot, red);
  tr = block_sum(tr, red);
  double* res = A.result;  // [d var, d l (Q), d Z (M Q), d beta]
  for (int e = threadIdx.x; e < mq; e += blockDim.x) {
    const int a = e % m, j = e / m;
    const double il2 = 1.0 / (A.ls[j] * A.ls[j]);
    res[1 + q + e] = 2.0 * (A.wz[e] - rs[a] * A.z[e]) * il2;
  }
  // sum_ab W_ab (z_a - z_b)^2 = 2 (sum_a rs_a z_a^2 - z^T W z) per dimension (a warp per q, fixed tree)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < q; j += blockDim.x >> 5) {
    double s2 = 0.0, cross = 0.0;
    for (int a = lane; a < m; a += 32) {
      const double za = A.z[a + j * m];
      s2 += rs[a] * za * za;
      cross += za * A.wz[a + j * m];
    }
    s2 = dev_warp_sum(s2);
    cross = dev_warp_sum(cross);
    if (lane == 0) res[1 + j] = 2.0 * (s2 - cross) / (A.ls[j] * A.ls[j] * A.ls[j]);
  }
  if (threadIdx.x == 0) {
    const double* sc = A.sc;
    const double nd = double(A.n), yy = A.packed[1], phi0 = A.packed[0];
    res[0] = tot / A.var + sc[kScJitterFactor] * tr;
    res[1 + q + mq] = 0.5 * dd * nd / beta - 0.5 * dd * sc[kScAp] - 0.5 * yy + beta * sc[kScPg] -
                      0.5 * beta * beta * tg - 0.5 * dd * phi0 + 0.5 * dd * sc[kScKp];
  }
}

// final gradient vector = the coordinator's terms (deferred_small_kernel) + the psi gradients
__global__ void finish_add_kernel(double* __restrict__ res, const double* __restrict__ pgrads, int count) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) res[e] += pgrads[e];
}

__global__ void init_status_kernel(double* sc, const int* info_k) {
  if (threadIdx.x == 0) sc[kScStatusK] = info_k[0] ? double(kStGramFailed) : 0.0;
}
// this evaluation's status: the prefactor's, plus A's factorisation
__global__ void status_a_kernel(double* sc, const int* info_a) {
  if (threadIdx.x == 0) sc[kScStatus] = double(int(sc[kScStatusK]) | (info_a[0] ? kStAFailed : 0));
}

inline unsigned blocks_for(int64_t n) { return unsigned((n + 255) / 256); }

}  // namespace

int64_t dc_workspace_doubles(int m, int q, int d) {
  const int64_t mm = int64_t(m) * m, md = int64_t(m) * std::max(d, 1), mq = int64_t(m) * q;
  // kmm lk wk kinv a la wa ainv phi ggt tmp kpk dkmm w (14 M x M), g phig (M x D), rs (M), wz (M x Q),
  // scalars, result, ls (Q), info (2 ints in 1 double)
  return 14 * mm + 2 * md + m + mq + kScCount + (2 + q + mq) + q + 2;
}

void dc_bind(DcArgs& A, double* ws) {
  const int m = A.m, q = A.q;
  const int64_t mm = int64_t(m) * m, md = int64_t(m) * std::max(A.d, 1), mq = int64_t(m) * q;
  double* p = ws;
  auto take = [&p](int64_t n) {
    double* r = p;
    p += n;
    return r;
  };
  A.kmm = take(mm);
  A.lk = take(mm);
  A.wk = take(mm);
  A.kinv = take(mm);
  A.a = take(mm);
  A.la = take(mm);
  A.wa = take(mm);
  A.ainv = take(mm);
  A.phi = take(mm);
  A.ggt = take(mm);
  A.tmp = take(mm);
  A.kpk = take(mm);
  A.dkmm = take(mm);
  A.w = take(mm);
  A.g = take(md);
  A.phig = take(md);
  A.rs = take(m);
  A.wz = take(mq);
  A.sc = take(kScCount);
  A.result = take(2 + q + mq);
  A.ls = take(q);  // uploaded by the caller
  A.info = reinterpret_cast<int*>(take(2));
}

size_t small_smem(int m) { return sizeof(double) * 2 * size_t(m) * m; }

namespace {
struct LsArg {
  double v[64];
};
__global__ void upload_ls_kernel(double* __restrict__ dst, int q, const LsArg ls) {
  if (threadIdx.x < q) dst[threadIdx.x] = ls.v[threadIdx.x];
}
}  // namespace

int dc_upload_ls(const DcArgs& A, const double* ls, cudaStream_t st) {
  if (A.q > 64) return 1;
  LsArg a{};
  for (int i = 0; i < A.q; ++i) a.v[i] = ls[i];
  upload_ls_kernel<<<1, 64, 0, st>>>(const_cast<double*>(A.ls), A.q, a);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int dc_prefactor(const DcArgs& A, cudaStream_t st) {
  const int m = A.m;
  if (m <= kSmallM) {
    if (cudaFuncSetAttribute(prefactor_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(small_smem(kSmallM))) != cudaSuccess)
      return 3;
    prefactor_small_kernel<<<1, 1024, small_smem(m), st>>>(A);
    g_tc_launches.fetch_add(1);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  gram_kernel<<<blocks_for(int64_t(m) * m), 256, 0, st>>>(A.z, m, A.q, A.ls, A.var, A.kmm);
  g_tc_launches.fetch_add(1);
  if (dla::cholesky(A.kmm, m, A.lk, 0, A.jitter_factor, A.var, A.sc + kScLogDetK, A.info, st)) return 3;
  init_status_kernel<<<1, 32, 0, st>>>(A.sc, A.info);
  g_tc_launches.fetch_add(1);
  if (dla::trinv(A.lk, m, A.wk, st)) return 3;
  if (dla::gemm(true, false, m, m, m, 1.0, A.wk, m, A.wk, m, 0.0, A.kinv, m, st)) return 3;
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int dc_bound(const DcArgs& A, float* u, float* dpsi, double* u64, double* dpsi64, cudaStream_t st) {
  const int m = A.m, d = A.d;
  if (m <= kSmallM) {
    if (cudaFuncSetAttribute(bound_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(small_smem(kSmallM))) != cudaSuccess)
      return 3;
    bound_small_kernel<<<1, 1024, small_smem(m), st>>>(A, u, dpsi, u64, dpsi64);
    g_tc_launches.fetch_add(1);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  const int64_t mm = int64_t(m) * m;
  build_a_kernel<<<blocks_for(mm), 256, 0, st>>>(A.kmm, A.packed, m, A.beta, A.var, A.sc, A.a);
  unpack_phi_kernel<<<blocks_for(mm), 256, 0, st>>>(A.packed, m, A.phi);
  g_tc_launches.fetch_add(2);
  if (dla::cholesky(A.a, m, A.la, 1, 0.0, 0.0, A.sc + kScLogDetA, A.info + 1, st)) return 3;
  status_a_kernel<<<1, 32, 0, st>>>(A.sc, A.info + 1);
  g_tc_launches.fetch_add(1);
  if (dla::trinv(A.la, m, A.wa, st)) return 3;
  if (dla::gemm(true, false, m, m, m, 1.0, A.wa, m, A.wa, m, 0.0, A.ainv, m, st)) return 3;
  const double* psi = A.packed + 4 + int64_t(m) * (m + 1) / 2;
  if (dla::gemm(false, false, m, d, m, 1.0, A.ainv, m, psi, m, 0.0, A.g, m, st)) return 3;
  if (dla::gemm(false, true, m, m, d, 1.0, A.g, m, A.g, m, 0.0, A.ggt, m, st)) return 3;
  bound_kernel<<<1, 1024, 0, st>>>(A);
  const int64_t na = std::max<int64_t>(int64_t(A.mv) * A.mv, int64_t(std::max(d, 1)) * A.mv);
  adjoint_kernel<<<blocks_for(na), 256, 0, st>>>(A, u, dpsi, u64, dpsi64);
  g_tc_launches.fetch_add(2);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int dc_bound_split(const DcArgs& A, float* u, float* dpsi, double* u64, double* dpsi64, cudaStream_t st,
                   cudaStream_t side, cudaStream_t side2, cudaEvent_t* ev) {
  const int m = A.m;
  if (m > kSmallM || !side || !side2) {  // one stream: the whole coordinator before the backward
    if (int rc = dc_bound(A, u, dpsi, u64, dpsi64, st)) return rc;
    if (int rc = dc_deferred(A, st)) return rc;
    if (cudaEventRecord(ev[0], st) != cudaSuccess || cudaEventRecord(ev[1], st) != cudaSuccess) return 3;
    return 0;
  }
  const int smax = int(small_smem(kSmallM));
  if (cudaFuncSetAttribute(bound_g_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(g_small_smem(kSmallM))) != cudaSuccess ||
      cudaFuncSetAttribute(bound_u_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smax) != cudaSuccess ||
      cudaFuncSetAttribute(deferred_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smax) != cudaSuccess)
    return 3;
  // side2: Kmm^-1 Phi Kmm^-1 from the statistics alone, concurrently with K1
  if (cudaEventRecord(ev[2], st) != cudaSuccess || cudaStreamWaitEvent(side2, ev[2], 0) != cudaSuccess) return 3;
  deferred_small_kernel<<<1, 1024, small_smem(m), side2>>>(A, 1);
  if (cudaEventRecord(ev[3], side2) != cudaSuccess) return 3;
  bound_g_small_kernel<<<1, kG1Threads, g_small_smem(m), st>>>(A, dpsi, dpsi64);
  if (cudaEventRecord(ev[0], st) != cudaSuccess || cudaStreamWaitEvent(side, ev[0], 0) != cudaSuccess) return 3;
  bound_u_small_kernel<<<1, 1024, small_smem(m), side>>>(A, u, u64);
  if (cudaStreamWaitEvent(side, ev[3], 0) != cudaSuccess) return 3;
  deferred_small_kernel<<<1, 1024, small_smem(m), side>>>(A, 2);
  if (cudaEventRecord(ev[1], side) != cudaSuccess) return 3;
  g_tc_launches.fetch_add(4);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int dc_deferred(const DcArgs& A, cudaStream_t st) {
  const int m = A.m, d = A.d;
  if (m <= kSmallM) {
    if (cudaFuncSetAttribute(deferred_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(small_smem(kSmallM))) != cudaSuccess)
      return 3;
    deferred_small_kernel<<<1, 1024, small_smem(m), st>>>(A, 0);
    g_tc_launches.fetch_add(1);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  if (dla::gemm(false, false, m, m, m, 1.0, A.kinv, m, A.phi, m, 0.0, A.tmp, m, st)) return 3;
  if (dla::gemm(false, false, m, m, m, 1.0, A.tmp, m, A.kinv, m, 0.0, A.kpk, m, st)) return 3;
  if (dla::gemm(false, false, m, d, m, 1.0, A.phi, m, A.g, m, 0.0, A.phig, m, st)) return 3;
  dkmm_kernel<<<blocks_for(int64_t(m) * m), 256, 0, st>>>(A);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int dc_finish(const DcArgs& A, const double* pgrads, cudaStream_t st) {
  const int m = A.m;
  if (m <= kSmallM) {  // deferred_small_kernel formed the rest of the assembly
    finish_add_kernel<<<1, 256, 0, st>>>(A.result, pgrads, 1 + A.q + m * A.q);
    g_tc_launches.fetch_add(1);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  w_kernel<<<blocks_for(int64_t(m) * m), 256, 0, st>>>(A);
  rowsum_kernel<<<(m + 127) / 128, 128, 0, st>>>(A);
  g_tc_launches.fetch_add(2);
  if (dla::gemm(false, false, m, A.q, m, 1.0, A.w, m, A.z, m, 0.0, A.wz, m, st)) return 3;
  finish_kernel<<<1, 1024, 0, st>>>(A, pgrads);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// ---- prediction (predict_from_cache, model.hpp:197-217) ----
namespace {
__global__ void kstar_kernel(const double* __restrict__ xs, int64_t t, const double* __restrict__ z, int m, int q,
                             const double* __restrict__ ls, double var, double* __restrict__ ks) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= t * m) return;
  const int64_t r = e % t;
  const int a = int(e / t);
  double d2 = 0.0;
  for (int j = 0; j < q; ++j) {
    const double dd = (xs[r + j * t] - z[a + int64_t(j) * m]) / ls[j];
    d2 += dd * dd;
  }
  ks[e] = var * exp(-0.5 * d2);
}

// var = variance - |L_k^-1 k*|^2 + |L_a^-1 k*|^2, floored at 1e-15 variance, + 1/beta (observation);
// the same column for every output dimension.
__global__ void pred_var_kernel(const double* __restrict__ v1, const double* __restrict__ v2, int64_t t, int m, int d,
                                double var, double beta, int obs, double* __restrict__ out) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= t) return;
  double n1 = 0.0, n2 = 0.0;
  for (int i = 0; i < m; ++i) {
    const double a = v1[r + int64_t(i) * t], b = v2[r + int64_t(i) * t];
    n1 += a * a;
    n2 += b * b;
  }
  double v = fmax(var - n1 + n2, 1e-15 * var);
  if (obs) v += 1.0 / beta;
  for (int c = 0; c < d; ++c) out[r + int64_t(c) * t] = v;
}
}  // namespace

extern "C" int sgpx_debug_dc_profile(long long* host16) {
  long long* d = nullptr;
  if (cudaMalloc(&d, 16 * sizeof(long long)) != cudaSuccess) return 3;
  dc_prof_kernel<<<1, 32>>>(d);
  cudaMemcpy(host16, d, 16 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return 0;
}

int64_t dc_predict_doubles(int64_t t, int m, int q, int d) { return t * (q + 3 * int64_t(m) + 2 * int64_t(d)) + 8; }

int dc_predict(const DcArgs& A, const double* xs, int64_t t, int obs, double* work, double* mean, double* var,
               cudaStream_t st) {
  const int m = A.m, q = A.q, d = A.d;
  double* ks = work;
  double* v1 = ks + t * m;
  double* v2 = v1 + t * m;
  kstar_kernel<<<unsigned((t * m + 255) / 256), 256, 0, st>>>(xs, t, A.z, m, q, A.ls, A.var, ks);
  g_tc_launches.fetch_add(1);
  if (dla::gemm(false, false, int(t), d, m, A.beta, ks, t, A.g, m, 0.0, mean, t, st)) return 3;
  if (dla::gemm(false, true, int(t), m, m, 1.0, ks, t, A.wk, m, 0.0, v1, t, st)) return 3;
  if (dla::gemm(false, true, int(t), m, m, 1.0, ks, t, A.wa, m, 0.0, v2, t, st)) return 3;
  pred_var_kernel<<<unsigned((t + 255) / 256), 256, 0, st>>>(v1, v2, t, m, d, A.var, A.beta, obs, var);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace sgpx
