// coordinator.cpp -- fp64 M x M algebra of Engine::evaluate (see coordinator.hpp).
#include "coordinator.hpp"

#include <algorithm>
#include <cmath>

namespace sgpx {
namespace coord {

void Kernel::validate() const {  // kernels.hpp:18-24
  require(std::isfinite(variance) && variance > 0.0, "kernel variance must be positive");
  require(!ls.empty(), "kernel needs at least one lengthscale");
  for (double l : ls) require(std::isfinite(l) && l > 0.0, "kernel lengthscales must be positive");
}

// Left-looking Cholesky on column-major storage, inner loops over contiguous
// column entries (vectorisable).  Works on a copy so A is untouched.
bool cholesky(const Mat& a, Mat& L) {
  const int64_t n = a.r;
  L = a;
  for (int64_t j = 0; j < n; ++j) {
    double* cj = L.col(j);
    // cj[j:n] -= sum_k L[j:n, k] * L[j, k]
    for (int64_t k = 0; k < j; ++k) {
      const double ljk = L(j, k);
      const double* ck = L.col(k);
      for (int64_t i = j; i < n; ++i) cj[i] -= ck[i] * ljk;
    }
    const double djj = cj[j];
    if (!(djj > 0.0)) return false;
    const double ljj = std::sqrt(djj);
    const double inv = 1.0 / ljj;
    cj[j] = ljj;
    for (int64_t i = j + 1; i < n; ++i) cj[i] *= inv;
    for (int64_t i = 0; i < j; ++i) cj[i] = 0.0;
  }
  return true;
}

double log_det_chol(const Mat& L) {
  double s = 0.0;
  for (int64_t i = 0; i < L.r; ++i) s += std::log(L(i, i));
  return 2.0 * s;
}

void chol_solve(const Mat& L, Mat& B) {
  const int64_t n = L.r;
  for (int64_t c = 0; c < B.c; ++c) {
    double* x = B.col(c);
    // forward: L y = b (column-oriented)
    for (int64_t k = 0; k < n; ++k) {
      x[k] /= L(k, k);
      const double xk = x[k];
      const double* lk = L.col(k);
      for (int64_t i = k + 1; i < n; ++i) x[i] -= lk[i] * xk;
    }
    // backward: L^T x = y (dot-product oriented on columns of L)
    for (int64_t k = n - 1; k >= 0; --k) {
      const double* lk = L.col(k);
      double s = x[k];
      for (int64_t i = k + 1; i < n; ++i) s -= lk[i] * x[i];
      x[k] = s / lk[k];
    }
  }
}

static Mat transpose(const Mat& a) {
  Mat t(a.c, a.r);
  for (int64_t j = 0; j < a.c; ++j)
    for (int64_t i = 0; i < a.r; ++i) t(j, i) = a(i, j);
  return t;
}

// C = A B (column-major), 8 x 4 register blocks of C (GCC vector types, AVX2 with
// -march=x86-64-v3) accumulated over p in ascending order: each element's summation order is
// fixed, so results are bitwise reproducible.
typedef double v4d __attribute__((vector_size(32)));
static inline v4d load4(const double* p) {
  v4d v;
  __builtin_memcpy(&v, p, sizeof(v));
  return v;
}
static inline void store4(double* p, v4d v) { __builtin_memcpy(p, &v, sizeof(v)); }

static void gemm_nn(const Mat& A, const Mat& B, Mat& C) {
  const int64_t m = A.r, k = A.c, n = B.c;
  const double* __restrict__ a = A.v.data();
  const double* __restrict__ b = B.v.data();
  double* __restrict__ c = C.v.data();
  int64_t j0 = 0;
  for (; j0 + 4 <= n; j0 += 4) {
    int64_t i0 = 0;
    for (; i0 + 8 <= m; i0 += 8) {
      v4d c00 = {0, 0, 0, 0}, c01 = c00, c10 = c00, c11 = c00, c20 = c00, c21 = c00, c30 = c00, c31 = c00;
      const double* b0 = b + j0 * k;
      for (int64_t p = 0; p < k; ++p) {
        const v4d a0 = load4(a + p * m + i0), a1 = load4(a + p * m + i0 + 4);
        const double s0 = b0[p], s1 = b0[k + p], s2 = b0[2 * k + p], s3 = b0[3 * k + p];
        c00 += a0 * s0;
        c01 += a1 * s0;
        c10 += a0 * s1;
        c11 += a1 * s1;
        c20 += a0 * s2;
        c21 += a1 * s2;
        c30 += a0 * s3;
        c31 += a1 * s3;
      }
      store4(c + j0 * m + i0, c00);
      store4(c + j0 * m + i0 + 4, c01);
      store4(c + (j0 + 1) * m + i0, c10);
      store4(c + (j0 + 1) * m + i0 + 4, c11);
      store4(c + (j0 + 2) * m + i0, c20);
      store4(c + (j0 + 2) * m + i0 + 4, c21);
      store4(c + (j0 + 3) * m + i0, c30);
      store4(c + (j0 + 3) * m + i0 + 4, c31);
    }
    for (; i0 < m; ++i0) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int64_t p = 0; p < k; ++p)
        for (int jj = 0; jj < 4; ++jj) acc[jj] += a[p * m + i0] * b[(j0 + jj) * k + p];
      for (int jj = 0; jj < 4; ++jj) c[(j0 + jj) * m + i0] = acc[jj];
    }
  }
  for (; j0 < n; ++j0)
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) acc += a[p * m + i] * b[j0 * k + p];
      c[j0 * m + i] = acc;
    }
}

Mat gemm(const Mat& A, bool ta, const Mat& B, bool tb) {
  const int64_t m = ta ? A.c : A.r, n = tb ? B.r : B.c;
  Mat C(m, n);
  if (ta && tb) gemm_nn(transpose(A), transpose(B), C);
  else if (ta) gemm_nn(transpose(A), B, C);
  else if (tb) gemm_nn(A, transpose(B), C);
  else gemm_nn(A, B, C);
  return C;
}

static void symmetrize(Mat& a) {
  for (int64_t j = 0; j < a.c; ++j)
    for (int64_t i = j + 1; i < a.r; ++i) {
      const double s = 0.5 * (a(i, j) + a(j, i));
      a(i, j) = s;
      a(j, i) = s;
    }
}

Mat chol_inverse(const Mat& L) {
  // W = L^{-1} (lower triangular, column-oriented forward substitution), then
  // (L L^T)^{-1} = W^T W computed as dot products of W's columns (exactly symmetric).
  const int64_t n = L.r;
  Mat W(n, n);
  for (int64_t j = 0; j < n; ++j) {
    double* x = W.col(j);
    x[j] = 1.0;
    for (int64_t k = j; k < n; ++k) {
      x[k] /= L(k, k);
      const double xk = x[k];
      const double* lk = L.col(k);
      for (int64_t i = k + 1; i < n; ++i) x[i] -= lk[i] * xk;
    }
  }
  Mat X(n, n);
  for (int64_t j = 0; j < n; ++j) {
    const double* wj = W.col(j);
    for (int64_t i = j; i < n; ++i) {
      const double* wi = W.col(i);
      // rows k >= max(i, j) = i; four vector accumulators over k in a fixed order
      int64_t k = i;
      v4d a0 = {0, 0, 0, 0}, a1 = a0, a2 = a0, a3 = a0;
      for (; k + 16 <= n; k += 16) {
        a0 += load4(wi + k) * load4(wj + k);
        a1 += load4(wi + k + 4) * load4(wj + k + 4);
        a2 += load4(wi + k + 8) * load4(wj + k + 8);
        a3 += load4(wi + k + 12) * load4(wj + k + 12);
      }
      for (; k + 4 <= n; k += 4) a0 += load4(wi + k) * load4(wj + k);
      const v4d t = (a0 + a1) + (a2 + a3);
      double s = (t[0] + t[1]) + (t[2] + t[3]);
      for (; k < n; ++k) s += wi[k] * wj[k];
      X(i, j) = s;
      X(j, i) = s;
    }
  }
  return X;
}

Mat kern_gram(const Mat& z, const Kernel& k, double jitter, bool* near_dup) {
  k.validate();
  require(z.c == k.q(), "kern_gram Z: column count does not match kernel input dimension");
  for (double x : z.v) require(std::isfinite(x), "kern_gram Z: non-finite entries");
  require(z.r >= 1, "kern_gram: need at least one inducing input");
  require(jitter >= 0.0, "kern_gram: jitter must be non-negative");
  const int64_t m = z.r, q = z.c;
  std::vector<double> il2(q);
  for (int64_t j = 0; j < q; ++j) il2[j] = 1.0 / (k.ls[j] * k.ls[j]);
  Mat out(m, m);
  bool dup = false;
  for (int64_t a = 0; a < m; ++a) {
    out(a, a) = k.variance + jitter;
    for (int64_t b = a + 1; b < m; ++b) {
      double d2 = 0.0;
      for (int64_t j = 0; j < q; ++j) {
        const double d = z(a, j) - z(b, j);
        d2 += d * d * il2[j];
      }
      if (d2 < 1e-24) dup = true;
      const double v = k.variance * std::exp(-0.5 * d2);
      out(a, b) = v;
      out(b, a) = v;
    }
  }
  if (near_dup) *near_dup = dup;
  return out;
}

GramFactor factor_gram(const Mat& z, const Kernel& k, double jitter_factor) {
  require(jitter_factor >= 0.0, "factor_gram: jitter factor must be non-negative");
  double jf = jitter_factor;
  for (;;) {
    GramFactor f;
    f.jitter_factor = jf;
    f.jitter = jf * k.variance;
    f.kmm = kern_gram(z, k, f.jitter, nullptr);
    if (cholesky(f.kmm, f.L)) {
      f.log_det = log_det_chol(f.L);
      return f;
    }
    if (jf >= 1e-2)
      throw NumericError(
          "factor_gram: Gram matrix not factorizable even at jitter 1e-2 * variance (ill-conditioned inducing "
          "inputs)");
    jf = (jf == 0.0) ? 1e-6 : jf * 10.0;
  }
}

// bound.hpp:52-62: escalating diagonal shift anchored to the matrix's own scale.
static bool factor_spd(const Mat& a, Mat& L) {
  if (cholesky(a, L)) return true;
  double scale = 0.0;
  for (int64_t i = 0; i < a.r; ++i) scale = std::max(scale, std::fabs(a(i, i)));
  for (double f = 1e-10; f <= 1e-2; f *= 10.0) {
    Mat b = a;
    for (int64_t i = 0; i < a.r; ++i) b(i, i) += f * scale;
    if (cholesky(b, L)) return true;
  }
  return false;
}

Stats unpack_stats(const double* p, int64_t m, int64_t d) {
  Stats s;
  s.phi = p[0];
  s.yy = p[1];
  s.n = p[2];
  s.kl = p[3];
  s.phi_big = Mat(m, m);
  const double* pairs = p + 4;
  int64_t idx = 0;
  for (int64_t a = 0; a < m; ++a)
    for (int64_t b = a; b < m; ++b) {
      const double v = pairs[idx++];
      s.phi_big(a, b) = v;
      s.phi_big(b, a) = v;
    }
  s.psi_y = Mat(m, d);
  std::copy(pairs + idx, pairs + idx + m * d, s.psi_y.v.begin());
  return s;
}

Prefactor prefactor(const Mat& z, const Kernel& k, double jitter_factor) {
  Prefactor p;
  p.gram = factor_gram(z, k, jitter_factor);
  p.kmm_inv = chol_inverse(p.gram.L);
  return p;
}

Result coordinate(bool latent, int64_t n, int64_t d, const Stats& st, const Mat& z, const Kernel& k, double beta,
                  double jitter_factor, bool with_adjoints, bool defer_host_only, const Prefactor* pre) {
  const int64_t m = z.r;
  require(beta > 0.0 && std::isfinite(beta), "bound: beta must be positive");
  require(n >= 1 && d >= 1, "bound: need N >= 1 and D >= 1");
  require(int64_t(st.n) == n, "bound: stats n_count does not match N");
  require(st.phi >= 0.0 && st.yy >= 0.0, "bound: phi and yy must be non-negative");
  Result r;
  r.gram = pre ? pre->gram : factor_gram(z, k, jitter_factor);
  // bound_core (bound.hpp:84-119).  The Kmm factor of factor_gram is exactly
  // factor_spd(Kmm)'s first (successful) attempt.
  const Mat& Lk = r.gram.L;
  const double log_det_kmm = r.gram.log_det;
  Mat a = r.gram.kmm;
  for (size_t i = 0; i < a.v.size(); ++i) a.v[i] += beta * st.phi_big.v[i];
  Mat La;
  if (!factor_spd(a, La)) throw NumericError("bound (Kmm + beta*Phi): Cholesky factorization failed after jitter escalation");
  const double log_det_a = log_det_chol(La);
  const Mat a_inv = chol_inverse(La);
  const Mat g = gemm(a_inv, false, st.psi_y, false);
  const Mat kmm_inv = pre ? pre->kmm_inv : chol_inverse(Lk);
  const double log_2pi = 1.8378770664093454835606594728112;
  const double nd = double(n), dd = double(d);
  Breakdown& bd = r.bd;
  bd.log_det = dd * (0.5 * nd * std::log(beta) + 0.5 * log_det_kmm - 0.5 * nd * log_2pi - 0.5 * log_det_a);
  bd.data_fit = -0.5 * beta * st.yy;
  double pg = 0.0;
  for (size_t i = 0; i < g.v.size(); ++i) pg += st.psi_y.v[i] * g.v[i];
  bd.quadratic = 0.5 * beta * beta * pg;
  bd.trace_phi = -0.5 * beta * dd * st.phi;
  double kp = 0.0, ap = 0.0;
  for (size_t i = 0; i < kmm_inv.v.size(); ++i) {
    kp += kmm_inv.v[i] * st.phi_big.v[i];
    ap += a_inv.v[i] * st.phi_big.v[i];
  }
  bd.trace_kmm = 0.5 * beta * dd * kp;
  bd.kl = latent ? -st.kl : 0.0;
  bd.total = bd.sum();
  if (!std::isfinite(bd.total)) throw NumericError("bound: non-finite value");
  if (!with_adjoints) return r;

  // adjoints_from_core (bound.hpp:196-226)
  Adjoints& adj = r.adj;
  adj.d_phi = -0.5 * beta * dd;
  adj.d_psi_y = g;
  for (double& x : adj.d_psi_y.v) x *= beta * beta;
  Mat ggt = gemm(g, false, g, true);
  symmetrize(ggt);
  adj.d_phi_big = Mat(m, m);
  for (size_t i = 0; i < ggt.v.size(); ++i)
    adj.d_phi_big.v[i] = -0.5 * beta * dd * a_inv.v[i] - 0.5 * beta * beta * beta * ggt.v[i] + 0.5 * beta * dd * kmm_inv.v[i];
  r.kmm_inv = kmm_inv;
  r.a_inv = a_inv;
  r.g = g;
  r.ggt = ggt;
  r.ap = ap;
  r.kp = kp;
  r.pg = pg;
  r.deferred = true;
  if (!defer_host_only) complete_adjoints(r, st, n, d, beta);
  return r;
}

void complete_adjoints(Result& r, const Stats& st, int64_t n, int64_t d, double beta) {
  if (!r.deferred) return;
  const int64_t m = r.g.r;
  const double nd = double(n), dd = double(d);
  const Mat& kmm_inv = r.kmm_inv;
  const Mat& a_inv = r.a_inv;
  const Mat& g = r.g;
  const Mat& ggt = r.ggt;
  Adjoints& adj = r.adj;
  Mat kpk = gemm(gemm(kmm_inv, false, st.phi_big, false), false, kmm_inv, false);
  symmetrize(kpk);
  adj.d_kmm = Mat(m, m);
  for (size_t i = 0; i < ggt.v.size(); ++i)
    adj.d_kmm.v[i] = 0.5 * dd * kmm_inv.v[i] - 0.5 * dd * a_inv.v[i] - 0.5 * beta * beta * ggt.v[i] - 0.5 * beta * dd * kpk.v[i];
  const Mat phig = gemm(st.phi_big, false, g, false);
  double tr_gphig = 0.0;
  for (size_t i = 0; i < g.v.size(); ++i) tr_gphig += g.v[i] * phig.v[i];
  // d_beta: the sum of the workers' beta_share (parallel.hpp:185-195) equals this
  // global expression (bound.hpp:217-223) evaluated on the reduced statistics.
  adj.d_beta = 0.5 * dd * nd / beta - 0.5 * dd * r.ap - 0.5 * st.yy + beta * r.pg - 0.5 * beta * beta * tr_gphig -
               0.5 * dd * st.phi + 0.5 * dd * r.kp;
  r.deferred = false;
  r.kmm_inv = Mat();
  r.a_inv = Mat();
  r.g = Mat();
  r.ggt = Mat();
}

KernGrads kern_grads_zz(const Mat& z, const Kernel& k, const Mat& up) {
  // kern_grads(Z, Z, k, U) (kernels.hpp:124-164) with d_z + d_x summed, for a symmetric
  // upstream U = dL/dKmm.  With W = U o K (Hadamard), sum over both slots:
  //   d_z + d_x = 2 (W Z - diag(W 1) Z) / l^2,   d_l_q = sum_nm W_nm (z_nq - z_mq)^2 / l_q^3,
  //   d_variance = sum W / variance.
  const int64_t m = z.r, q = z.c;
  std::vector<double> il2(q);
  for (int64_t j = 0; j < q; ++j) il2[j] = 1.0 / (k.ls[j] * k.ls[j]);
  Mat zs(m, q);  // z / l
  for (int64_t j = 0; j < q; ++j)
    for (int64_t a = 0; a < m; ++a) zs(a, j) = z(a, j) / k.ls[j];
  Mat W(m, m);
  for (int64_t b = 0; b < m; ++b)
    for (int64_t a = b; a < m; ++a) {
      double d2 = 0.0;
      for (int64_t j = 0; j < q; ++j) {
        const double d = zs(a, j) - zs(b, j);
        d2 += d * d;
      }
      const double kv = k.variance * std::exp(-0.5 * d2);
      W(a, b) = up(a, b) * kv;
      W(b, a) = up(b, a) * kv;
    }
  KernGrads g;
  g.d_ls.assign(q, 0.0);
  std::vector<double> rs(m, 0.0);
  double tot = 0.0;
  for (int64_t b = 0; b < m; ++b)
    for (int64_t a = 0; a < m; ++a) {
      rs[a] += W(a, b);
      tot += W(a, b);
    }
  g.d_variance = tot / k.variance;
  const Mat WZ = gemm(W, false, z, false);  // M x Q
  g.d_z = Mat(m, q);
  for (int64_t j = 0; j < q; ++j) {
    double s2 = 0.0, cross = 0.0;
    for (int64_t a = 0; a < m; ++a) {
      g.d_z(a, j) = 2.0 * (WZ(a, j) - rs[a] * z(a, j)) * il2[j];
      s2 += rs[a] * z(a, j) * z(a, j);
      cross += z(a, j) * WZ(a, j);
    }
    // sum_ab W_ab (z_a - z_b)^2 = 2 (sum_a rs_a z_a^2 - z^T W z) for symmetric W
    g.d_ls[j] = 2.0 * (s2 - cross) * il2[j] / k.ls[j];
  }
  return g;
}

}  // namespace coord
}  // namespace sgpx
