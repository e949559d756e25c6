// =============================================================================
// sgp_oracle.cpp -- CPU ORACLE (test infrastructure, NOT product code).
//
// A plain-C++ (no Eigen) fp64 restatement of the reference's psi-statistics hot
// path, used ONLY by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs, as the checker and the CPU baseline.  The product path
// (paper_1410_4984_b200/) never links, loads or calls anything in this file.
//
// Restated reference code (all paths relative to /root/reference):
//   Rng (splitmix64 + Box-Muller)         proj/include/sgp/common.hpp:45-97
//   kern_cross / kern_gram / kern_grads   proj/include/sgp/kernels.hpp:56-78, 83-112, 124-164
//   factor_gram (jitter escalation)       proj/include/sgp/kernels.hpp:177-197
//   check_adjoints, pair enumeration      proj/include/sgp/psi_stats.hpp:75-97
//   detail::sweep_stats (fwd + bwd)       proj/include/sgp/psi_stats.hpp:108-326
//   psi1_expected                         proj/include/sgp/psi_stats.hpp:351-376
//   factor_spd, bound_core                proj/include/sgp/bound.hpp:52-119
//   kl_gaussian                           proj/include/sgp/bound.hpp:164-169
//   adjoints_from_core                    proj/include/sgp/bound.hpp:196-226
//   make_partition                        proj/include/sgp/parallel.hpp:28-41
//   Worker::pass / beta_share             proj/include/sgp/parallel.hpp:132-195
//   reduce_reports                        proj/include/sgp/parallel.hpp:222-258
//   Engine::evaluate / run_pass           proj/include/sgp/parallel.hpp:370-479
//
// Parity pinning: the reference cannot be compiled here (Eigen3 is absent, see
// DESIGN.md "Oracle"), so this restatement is pinned against the known-answer
// tests of proj/tests/test_kernels.cpp and SPEC.md (KATs, quadrature, finite
// differences) in tests/test_oracle.py.
//
// Loop structure mirrors the reference (m-block -> n-chunk -> m; pair-block ->
// n-chunk -> pair) so the summation order follows the reference's canonical
// tile order.  Eigen's SIMD exp is a Cephes-style Pade approximant; exp() here
// is libm's (both are correctly rounded to within ~1 ulp).
// =============================================================================
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <deque>
#include <functional>
#include <vector>

namespace oracle {

using Index = int64_t;

struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
static void require(bool c, const std::string& m) {
  if (!c) throw std::invalid_argument(m);
}

// Column-major dense matrix (owning), mirrors Eigen::MatrixXd storage.
struct Mat {
  Index r = 0, c = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(Index rows, Index cols, double fill = 0.0) : r(rows), c(cols), v(size_t(rows * cols), fill) {}
  double& operator()(Index i, Index j) { return v[size_t(i + j * r)]; }
  double operator()(Index i, Index j) const { return v[size_t(i + j * r)]; }
  double* col(Index j) { return v.data() + j * r; }
  const double* col(Index j) const { return v.data() + j * r; }
};

// Non-owning column-major view with leading dimension (Eigen::Ref with outer stride).
struct View {
  const double* p = nullptr;
  Index r = 0, c = 0, ld = 0;
  double operator()(Index i, Index j) const { return p[i + j * ld]; }
  const double* col(Index j) const { return p + j * ld; }
  View rows(Index b, Index len) const { return View{p + b, len, c, ld}; }
};
static View view(const Mat& m) { return View{m.v.data(), m.r, m.c, m.r}; }

static bool all_finite(const View& a) {
  for (Index j = 0; j < a.c; ++j)
    for (Index i = 0; i < a.r; ++i)
      if (!std::isfinite(a(i, j))) return false;
  return true;
}

struct Kernel {
  double variance = 1.0;
  std::vector<double> ls;
  Index q() const { return Index(ls.size()); }
  void validate() const {  // kernels.hpp:18-24
    require(std::isfinite(variance) && variance > 0.0, "kernel variance must be positive");
    require(!ls.empty(), "kernel needs at least one lengthscale");
    for (double l : ls) require(std::isfinite(l) && l > 0.0, "kernel lengthscales must be positive");
  }
};

struct Tiles {
  Index block_span = 64, thread_span = 1024;  // common.hpp:30-37
  void validate() const { require(block_span >= 1 && thread_span >= 1, "TileConfig spans must be >= 1"); }
};

// ---------------------------------------------------------------------------
// Rng: splitmix64 + Box-Muller, common.hpp:45-97
// ---------------------------------------------------------------------------
struct Rng {
  uint64_t state;
  double spare = 0.0;
  bool have = false;
  explicit Rng(uint64_t seed) : state(seed ? seed : 0x9e3779b97f4a7c15ull) {}
  uint64_t u64() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform() { return (double(u64() >> 11) + 1.0) * 0x1.0p-53; }
  double normal() {
    if (have) { have = false; return spare; }
    double u1 = uniform(), u2 = uniform();
    double rr = std::sqrt(-2.0 * std::log(u1)), a = 6.283185307179586476925286766559 * u2;
    spare = rr * std::sin(a);
    have = true;
    return rr * std::cos(a);
  }
  uint64_t index(uint64_t n) {
    uint64_t limit = ~uint64_t{0} - (~uint64_t{0} % n), x = u64();
    while (x >= limit) x = u64();
    return x % n;
  }
};

// ---------------------------------------------------------------------------
// Kernels, kernels.hpp
// ---------------------------------------------------------------------------
static void check_inputs(const View& x, const Kernel& k, const char* name) {
  require(x.c == k.q(), std::string(name) + ": column count does not match kernel input dimension");
  require(all_finite(x), std::string(name) + ": non-finite entries");
}

static Mat kern_cross(const View& x, const View& z, const Kernel& k) {
  k.validate();
  check_inputs(x, k, "kern_cross X");
  check_inputs(z, k, "kern_cross Z");
  const Index n = x.r, m = z.r, q = k.q();
  std::vector<double> il2(q);
  for (Index j = 0; j < q; ++j) il2[j] = 1.0 / (k.ls[j] * k.ls[j]);
  Mat out(n, m);
  for (Index mm = 0; mm < m; ++mm)
    for (Index nn = 0; nn < n; ++nn) {
      double d2 = 0.0;
      for (Index j = 0; j < q; ++j) {
        double d = x(nn, j) - z(mm, j);
        d2 += d * d * il2[j];
      }
      out(nn, mm) = k.variance * std::exp(-0.5 * d2);
    }
  return out;
}

static Mat kern_gram(const View& z, const Kernel& k, double jitter, bool* near_dup = nullptr) {
  k.validate();
  check_inputs(z, k, "kern_gram Z");
  require(z.r >= 1, "kern_gram: need at least one inducing input");
  require(jitter >= 0.0, "kern_gram: jitter must be non-negative");
  const Index m = z.r, q = k.q();
  std::vector<double> il2(q);
  for (Index j = 0; j < q; ++j) il2[j] = 1.0 / (k.ls[j] * k.ls[j]);
  Mat out(m, m);
  bool dup = false;
  for (Index a = 0; a < m; ++a) {
    out(a, a) = k.variance + jitter;
    for (Index b = a + 1; b < m; ++b) {
      double d2 = 0.0;
      for (Index j = 0; j < q; ++j) {
        double d = z(a, j) - z(b, j);
        d2 += d * d * il2[j];
      }
      if (d2 < 1e-24) dup = true;
      double val = k.variance * std::exp(-0.5 * d2);
      out(a, b) = val;
      out(b, a) = val;
    }
  }
  if (near_dup) *near_dup = dup;
  return out;
}

struct KernGrads {
  double d_variance = 0.0;
  std::vector<double> d_ls;
  Mat d_z, d_x;
};

static KernGrads kern_grads(const View& x, const View& z, const Kernel& k, const View& up) {
  k.validate();
  check_inputs(x, k, "kern_grads X");
  check_inputs(z, k, "kern_grads Z");
  require(up.r == x.r && up.c == z.r, "kern_grads: upstream shape must be N x M");
  const Index n = x.r, m = z.r, q = k.q();
  std::vector<double> il2(q), il3(q);
  for (Index j = 0; j < q; ++j) {
    double l = k.ls[j];
    il2[j] = 1.0 / (l * l);
    il3[j] = 1.0 / (l * l * l);
  }
  KernGrads g;
  g.d_ls.assign(q, 0.0);
  g.d_z = Mat(m, q);
  g.d_x = Mat(n, q);
  for (Index mm = 0; mm < m; ++mm)
    for (Index nn = 0; nn < n; ++nn) {
      double d2 = 0.0;
      for (Index j = 0; j < q; ++j) {
        double d = x(nn, j) - z(mm, j);
        d2 += d * d * il2[j];
      }
      double val = k.variance * std::exp(-0.5 * d2);
      double uv = up(nn, mm) * val;
      g.d_variance += uv / k.variance;
      for (Index j = 0; j < q; ++j) {
        double d = x(nn, j) - z(mm, j);
        g.d_x(nn, j) -= uv * d * il2[j];
        g.d_z(mm, j) += uv * d * il2[j];
        g.d_ls[j] += uv * d * d * il3[j];
      }
    }
  return g;
}

// Lower Cholesky in place (Eigen LLT semantics: fail when a pivot is <= 0 or NaN).
static bool llt(const Mat& a, Mat& L) {
  const Index n = a.r;
  L = Mat(n, n);
  for (Index j = 0; j < n; ++j) {
    double d = a(j, j);
    for (Index k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
    if (!(d > 0.0)) return false;
    double ljj = std::sqrt(d);
    L(j, j) = ljj;
    for (Index i = j + 1; i < n; ++i) {
      double s = a(i, j);
      for (Index k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / ljj;
    }
  }
  return true;
}

static double log_det_llt(const Mat& L) {
  double s = 0.0;
  for (Index i = 0; i < L.r; ++i) s += std::log(L(i, i));
  return 2.0 * s;
}

// Solve (L L^T) X = B for column-major B (n x k).
static Mat llt_solve(const Mat& L, const Mat& B) {
  const Index n = L.r;
  Mat X = B;
  for (Index c = 0; c < B.c; ++c) {
    double* x = X.col(c);
    for (Index i = 0; i < n; ++i) {
      double s = x[i];
      for (Index k = 0; k < i; ++k) s -= L(i, k) * x[k];
      x[i] = s / L(i, i);
    }
    for (Index i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (Index k = i + 1; k < n; ++k) s -= L(k, i) * x[k];
      x[i] = s / L(i, i);
    }
  }
  return X;
}

static Mat identity(Index n) {
  Mat I(n, n);
  for (Index i = 0; i < n; ++i) I(i, i) = 1.0;
  return I;
}

static void symmetrize(Mat& a) {
  for (Index j = 0; j < a.c; ++j)
    for (Index i = j + 1; i < a.r; ++i) {
      double s = 0.5 * (a(i, j) + a(j, i));
      a(i, j) = s;
      a(j, i) = s;
    }
}

struct GramFactor {
  Mat kmm, L;
  double jitter = 0.0, jitter_factor = 0.0, log_det = 0.0;
};

static GramFactor factor_gram(const View& z, const Kernel& k, double jitter_factor) {
  require(jitter_factor >= 0.0, "factor_gram: jitter factor must be non-negative");
  double jf = jitter_factor;
  for (;;) {
    GramFactor f;
    f.jitter_factor = jf;
    f.jitter = jf * k.variance;
    f.kmm = kern_gram(z, k, f.jitter);
    if (llt(f.kmm, f.L)) {
      f.log_det = log_det_llt(f.L);
      return f;
    }
    if (jf >= 1e-2)
      throw NumericError(
          "factor_gram: Gram matrix not factorizable even at jitter 1e-2 * variance "
          "(ill-conditioned inducing inputs)");
    jf = (jf == 0.0) ? 1e-6 : jf * 10.0;
  }
}

// ---------------------------------------------------------------------------
// psi-statistics sweep, psi_stats.hpp:108-326
// ---------------------------------------------------------------------------
struct Stats {
  double phi = 0.0, yy = 0.0;
  Mat psi_y, phi_big;
  Index n_count = 0;
  static Stats zero(Index m, Index d) {
    Stats s;
    s.psi_y = Mat(m, d);
    s.phi_big = Mat(m, m);
    return s;
  }
  void add(const Stats& o) {
    phi += o.phi;
    for (size_t i = 0; i < psi_y.v.size(); ++i) psi_y.v[i] += o.psi_y.v[i];
    for (size_t i = 0; i < phi_big.v.size(); ++i) phi_big.v[i] += o.phi_big.v[i];
    yy += o.yy;
    n_count += o.n_count;
  }
};

struct Adj {
  double d_phi = 0.0;
  View d_psi_y, d_phi_big;
};

struct Grads {
  Mat d_mu, d_s, d_z;
  double d_variance = 0.0;
  std::vector<double> d_ls;
};

static void check_adjoints(const Adj& adj, Index m, Index d) {  // psi_stats.hpp:75-83
  require(adj.d_psi_y.r == m && adj.d_psi_y.c == d, "stats adjoints: d_psi_y shape must be M x D");
  require(adj.d_phi_big.r == m && adj.d_phi_big.c == m, "stats adjoints: d_phi_big shape must be M x M");
  double scale = 0.0, asym = 0.0;
  for (Index j = 0; j < m; ++j)
    for (Index i = 0; i < m; ++i) {
      scale = std::max(scale, std::fabs(adj.d_phi_big(i, j)));
      asym = std::max(asym, std::fabs(adj.d_phi_big(i, j) - adj.d_phi_big(j, i)));
    }
  require(asym <= 1e-10 * (1.0 + scale), "stats adjoints: d_phi_big must be symmetric");
}

static void pair_from_index(Index p, Index m, Index& m1, Index& m2) {  // psi_stats.hpp:88-97
  Index row = 0, row_start = 0;
  while (row_start + (m - row) <= p) {
    row_start += m - row;
    ++row;
  }
  m1 = row;
  m2 = row + (p - row_start);
}

static void sweep_stats(bool expected, const View& mu, const View& s, const View& y, const View& z,
                        const Kernel& kernel, const Tiles& tiles, const Adj* adj, Stats& stats,
                        Grads* grads) {
  kernel.validate();
  tiles.validate();
  const Index n = mu.r, q = mu.c, m = z.r, d = y.c;
  require(z.c == q, "stats sweep: Z column count mismatch");
  require(kernel.q() == q, "stats sweep: kernel dimension mismatch");
  require(y.r == n, "stats sweep: X/Y row counts differ");
  require(all_finite(mu) && all_finite(y) && all_finite(z), "stats sweep: non-finite data");
  if (expected) {
    for (Index j = 0; j < s.c; ++j)
      for (Index i = 0; i < s.r; ++i) require(s(i, j) > 0.0, "stats sweep: variances must be positive");
  }
  if (adj) check_adjoints(*adj, m, d);

  stats = Stats::zero(m, d);
  stats.phi = double(n) * kernel.variance;
  double yy = 0.0;
  for (Index j = 0; j < d; ++j)
    for (Index i = 0; i < n; ++i) yy += y(i, j) * y(i, j);
  stats.yy = yy;
  stats.n_count = n;

  if (grads) {
    grads->d_mu = expected ? Mat(n, q) : Mat();
    grads->d_s = expected ? Mat(n, q) : Mat();
    grads->d_z = Mat(m, q);
    grads->d_variance = adj ? adj->d_phi * double(n) : 0.0;
    grads->d_ls.assign(q, 0.0);
  }
  if (n == 0) return;

  const double var = kernel.variance;
  std::vector<double> l2(q), il2(q);
  for (Index j = 0; j < q; ++j) {
    l2[j] = kernel.ls[j] * kernel.ls[j];
    il2[j] = 1.0 / l2[j];
  }

  // Per-datapoint constants (psi_stats.hpp:144-167).
  std::vector<double> c1(n), c2(n);
  Mat iden1(n, q), iden2(n, q);
  if (expected) {
    std::vector<double> p1(n, 1.0), p2(n, 1.0);
    for (Index j = 0; j < q; ++j)
      for (Index i = 0; i < n; ++i) {
        p1[i] *= 1.0 + s(i, j) / l2[j];
        p2[i] *= 1.0 + 2.0 * s(i, j) / l2[j];
        iden1(i, j) = 1.0 / (s(i, j) + l2[j]);
        iden2(i, j) = 1.0 / (2.0 * s(i, j) + l2[j]);
      }
    for (Index i = 0; i < n; ++i) {
      c1[i] = var * (1.0 / std::sqrt(p1[i]));
      c2[i] = var * var * (1.0 / std::sqrt(p2[i]));
    }
  } else {
    for (Index i = 0; i < n; ++i) {
      c1[i] = var;
      c2[i] = var * var;
    }
    for (Index j = 0; j < q; ++j)
      for (Index i = 0; i < n; ++i) {
        iden1(i, j) = il2[j];
        iden2(i, j) = il2[j];
      }
  }

  const Index chunk = tiles.thread_span;
  std::vector<double> e(chunk), v(chunk), w(chunk), uv(chunk), t(chunk);

  // ---- psi part: blocks over inducing indices (psi_stats.hpp:172-219) ----
  for (Index mb = 0; mb < m; mb += tiles.block_span) {
    const Index mb_end = std::min(m, mb + tiles.block_span);
    for (Index nc = 0; nc < n; nc += chunk) {
      const Index len = std::min(chunk, n - nc);
      for (Index mm = mb; mm < mb_end; ++mm) {
        std::fill(e.begin(), e.begin() + len, 0.0);
        for (Index j = 0; j < q; ++j) {
          const double zj = z(mm, j);
          const double* muj = mu.col(j) + nc;
          const double* dj = iden1.col(j) + nc;
          for (Index i = 0; i < len; ++i) {
            double df = muj[i] - zj;
            e[i] += df * df * dj[i];
          }
        }
        for (Index i = 0; i < len; ++i) v[i] = c1[nc + i] * std::exp(-0.5 * e[i]);
        for (Index dd = 0; dd < d; ++dd) {
          const double* yd = y.col(dd) + nc;
          double acc = 0.0;
          for (Index i = 0; i < len; ++i) acc += v[i] * yd[i];
          stats.psi_y(mm, dd) += acc;
        }
        if (adj) {
          for (Index i = 0; i < len; ++i) {
            double acc = 0.0;
            for (Index dd = 0; dd < d; ++dd) acc += y(nc + i, dd) * adj->d_psi_y(mm, dd);
            w[i] = acc;
            uv[i] = w[i] * v[i];
          }
          double suv = 0.0;
          for (Index i = 0; i < len; ++i) suv += uv[i];
          grads->d_variance += suv / var;
          for (Index j = 0; j < q; ++j) {
            const double zj = z(mm, j);
            double dl = 0.0, dz = 0.0;
            for (Index i = 0; i < len; ++i) {
              double diff = mu(nc + i, j) - zj;
              double den = iden1(nc + i, j);
              double r = diff * den;
              if (expected) {
                grads->d_mu(nc + i, j) -= uv[i] * r;
                grads->d_s(nc + i, j) += uv[i] * 0.5 * den * (r * diff - 1.0);
                dl += uv[i] * kernel.ls[j] * den * (s(nc + i, j) * il2[j] + diff * r);
              } else {
                dl += uv[i] * diff * diff;
              }
              dz += uv[i] * r;
            }
            if (expected)
              grads->d_ls[j] += dl;
            else
              grads->d_ls[j] += dl * il2[j] / kernel.ls[j];
            grads->d_z(mm, j) += dz;
          }
        }
      }
    }
  }

  // ---- phi part: blocks over inducing index pairs (psi_stats.hpp:221-321) ----
  const Index pairs = m * (m + 1) / 2;
  const Index pb_span = tiles.block_span;
  std::vector<Index> pm1(pb_span), pm2(pb_span);
  std::vector<double> pconst(pb_span);
  Mat pzbar(pb_span, q);
  for (Index pb = 0; pb < pairs; pb += pb_span) {
    const Index pb_end = std::min(pairs, pb + pb_span), np = pb_end - pb;
    Index m1 = 0, m2 = 0;
    pair_from_index(pb, m, m1, m2);
    for (Index i = 0; i < np; ++i) {
      pm1[i] = m1;
      pm2[i] = m2;
      double a = 0.0;
      for (Index j = 0; j < q; ++j) {
        pzbar(i, j) = 0.5 * (z(m1, j) + z(m2, j));
        if (expected) {
          double dz = z(m1, j) - z(m2, j);
          a += dz * dz * il2[j] * 0.25;
        }
      }
      pconst[i] = expected ? std::exp(-a) : 1.0;
      if (++m2 == m) m2 = ++m1;
    }
    for (Index nc = 0; nc < n; nc += chunk) {
      const Index len = std::min(chunk, n - nc);
      for (Index i = 0; i < np; ++i) {
        const Index a = pm1[i], b = pm2[i];
        std::fill(e.begin(), e.begin() + len, 0.0);
        if (expected) {
          for (Index j = 0; j < q; ++j) {
            const double zb = pzbar(i, j);
            const double* muj = mu.col(j) + nc;
            const double* dj = iden2.col(j) + nc;
            for (Index k = 0; k < len; ++k) {
              double df = muj[k] - zb;
              e[k] += df * df * dj[k];
            }
          }
        } else {
          for (Index j = 0; j < q; ++j) {
            const double za = z(a, j), zb = z(b, j);
            const double* xj = mu.col(j) + nc;
            for (Index k = 0; k < len; ++k) {
              double da = xj[k] - za, db = xj[k] - zb;
              e[k] += 0.5 * il2[j] * (da * da + db * db);
            }
          }
        }
        double tile_sum = 0.0;
        for (Index k = 0; k < len; ++k) {
          v[k] = expected ? c2[nc + k] * pconst[i] * std::exp(-e[k]) : c2[nc + k] * std::exp(-e[k]);
          tile_sum += v[k];
        }
        stats.phi_big(a, b) += tile_sum;
        if (adj) {
          const double weight = (a == b) ? 1.0 : 2.0;
          const double u = adj->d_phi_big(a, b) * weight;
          if (u != 0.0) {
            double suv = 0.0;
            for (Index k = 0; k < len; ++k) {
              uv[k] = u * v[k];
              suv += uv[k];
            }
            grads->d_variance += 2.0 * suv / var;
            for (Index j = 0; j < q; ++j) {
              if (expected) {
                const double zbar = pzbar(i, j);
                const double dz12 = (z(a, j) - z(b, j)) * 0.5 * il2[j];
                const double cz = (z(a, j) - z(b, j)) * (z(a, j) - z(b, j)) * 0.5 * il2[j] * il2[j];
                double sa = 0.0, sb = 0.0, sl = 0.0;
                for (Index k = 0; k < len; ++k) {
                  double diffb = mu(nc + k, j) - zbar;
                  double den = iden2(nc + k, j);
                  double rb = diffb * den;
                  grads->d_mu(nc + k, j) -= 2.0 * uv[k] * rb;
                  grads->d_s(nc + k, j) += uv[k] * den * (2.0 * rb * diffb - 1.0);
                  sa += uv[k] * (rb - dz12);
                  sb += uv[k] * (rb + dz12);
                  sl += uv[k] * (2.0 * s(nc + k, j) * den * il2[j] + cz + 2.0 * rb * rb);
                }
                grads->d_z(a, j) += sa;
                grads->d_z(b, j) += sb;
                grads->d_ls[j] += kernel.ls[j] * sl;
              } else {
                const double za = z(a, j), zb = z(b, j);
                double sa = 0.0, sb = 0.0, sl = 0.0;
                for (Index k = 0; k < len; ++k) {
                  double xs = mu(nc + k, j);
                  double da = xs - za, db = xs - zb;
                  sa += uv[k] * da;
                  sb += uv[k] * db;
                  sl += uv[k] * (da * da + db * db);
                }
                grads->d_z(a, j) += sa * il2[j];
                grads->d_z(b, j) += sb * il2[j];
                grads->d_ls[j] += sl * il2[j] / kernel.ls[j];
              }
            }
          }
        }
      }
    }
  }
  for (Index a = 0; a < m; ++a)
    for (Index b = a + 1; b < m; ++b) stats.phi_big(b, a) = stats.phi_big(a, b);
}

// psi_stats.hpp:351-376
static Mat psi1_expected(const View& mu, const View& s, const View& z, const Kernel& kernel) {
  kernel.validate();
  require(mu.r == s.r && mu.c == s.c, "VariationalPosterior: mu and s shapes differ");
  require(all_finite(mu) && all_finite(s), "VariationalPosterior: non-finite entries");
  for (Index j = 0; j < s.c; ++j)
    for (Index i = 0; i < s.r; ++i) require(s(i, j) > 0.0, "VariationalPosterior: variances must be positive");
  require(z.c == mu.c, "psi1_expected: Z column count mismatch");
  require(kernel.q() == mu.c, "psi1_expected: kernel dimension mismatch");
  const Index n = mu.r, m = z.r, qd = mu.c;
  std::vector<double> c1(n, 1.0);
  Mat iden1(n, qd);
  for (Index j = 0; j < qd; ++j) {
    double l2 = kernel.ls[j] * kernel.ls[j];
    for (Index i = 0; i < n; ++i) {
      c1[i] *= 1.0 + s(i, j) / l2;
      iden1(i, j) = 1.0 / (s(i, j) + l2);
    }
  }
  for (Index i = 0; i < n; ++i) c1[i] = kernel.variance * (1.0 / std::sqrt(c1[i]));
  Mat out(n, m);
  for (Index mm = 0; mm < m; ++mm)
    for (Index i = 0; i < n; ++i) {
      double e = 0.0;
      for (Index j = 0; j < qd; ++j) {
        double df = mu(i, j) - z(mm, j);
        e += df * df * iden1(i, j);
      }
      out(i, mm) = c1[i] * std::exp(-0.5 * e);
    }
  return out;
}

// ---------------------------------------------------------------------------
// Bound, bound.hpp
// ---------------------------------------------------------------------------
static bool factor_spd(const Mat& a, Mat& L) {  // bound.hpp:52-62
  if (llt(a, L)) return true;
  double scale = 0.0;
  for (Index i = 0; i < a.r; ++i) scale = std::max(scale, std::fabs(a(i, i)));
  for (double f = 1e-10; f <= 1e-2; f *= 10.0) {
    Mat b = a;
    for (Index i = 0; i < a.r; ++i) b(i, i) += f * scale;
    if (llt(b, L)) return true;
  }
  return false;
}

struct Breakdown {
  double total = 0, log_det = 0, data_fit = 0, quadratic = 0, trace_phi = 0, trace_kmm = 0, kl = 0;
  double sum() const { return log_det + data_fit + quadratic + trace_phi + trace_kmm + kl; }
};

struct Core {
  Breakdown bd;
  Mat a, La, g, a_inv, kmm_inv, Lk;
  double log_det_a = 0, log_det_kmm = 0;
};

static Core bound_core(const Stats& st, const Mat& kmm, double beta, Index n, Index d) {
  require(beta > 0.0 && std::isfinite(beta), "bound: beta must be positive");
  require(n >= 1 && d >= 1, "bound: need N >= 1 and D >= 1");
  require(st.n_count == n, "bound: stats n_count does not match N");
  require(st.psi_y.c == d, "bound: stats D does not match D");
  require(kmm.r == kmm.c && kmm.r == st.psi_y.r, "bound: Kmm shape does not match stats");
  require(st.phi >= 0.0 && st.yy >= 0.0, "bound: phi and yy must be non-negative");
  const Index m = kmm.r;
  Core c;
  if (!factor_spd(kmm, c.Lk)) throw NumericError("bound (Kmm): Cholesky factorization failed after jitter escalation");
  c.log_det_kmm = log_det_llt(c.Lk);
  c.a = kmm;
  for (size_t i = 0; i < c.a.v.size(); ++i) c.a.v[i] += beta * st.phi_big.v[i];
  if (!factor_spd(c.a, c.La))
    throw NumericError("bound (Kmm + beta*Phi): Cholesky factorization failed after jitter escalation");
  c.log_det_a = log_det_llt(c.La);
  c.g = llt_solve(c.La, st.psi_y);
  c.a_inv = llt_solve(c.La, identity(m));
  symmetrize(c.a_inv);
  c.kmm_inv = llt_solve(c.Lk, identity(m));
  symmetrize(c.kmm_inv);
  const double log_2pi = 1.8378770664093454835606594728112;
  const double nd = double(n), dd = double(d);
  Breakdown& bd = c.bd;
  bd.log_det = dd * (0.5 * nd * std::log(beta) + 0.5 * c.log_det_kmm - 0.5 * nd * log_2pi - 0.5 * c.log_det_a);
  bd.data_fit = -0.5 * beta * st.yy;
  double pg = 0.0;
  for (size_t i = 0; i < st.psi_y.v.size(); ++i) pg += st.psi_y.v[i] * c.g.v[i];
  bd.quadratic = 0.5 * beta * beta * pg;
  bd.trace_phi = -0.5 * beta * dd * st.phi;
  double kp = 0.0;
  for (size_t i = 0; i < st.phi_big.v.size(); ++i) kp += c.kmm_inv.v[i] * st.phi_big.v[i];
  bd.trace_kmm = 0.5 * beta * dd * kp;
  bd.kl = 0.0;
  bd.total = bd.sum();
  if (!std::isfinite(bd.total)) throw NumericError("bound: non-finite value");
  return c;
}

static Mat matmul(const Mat& a, const Mat& b) {
  Mat c(a.r, b.c);
  for (Index j = 0; j < b.c; ++j)
    for (Index k = 0; k < a.c; ++k) {
      double bkj = b(k, j);
      for (Index i = 0; i < a.r; ++i) c(i, j) += a(i, k) * bkj;
    }
  return c;
}
static Mat transpose(const Mat& a) {
  Mat t(a.c, a.r);
  for (Index j = 0; j < a.c; ++j)
    for (Index i = 0; i < a.r; ++i) t(j, i) = a(i, j);
  return t;
}

struct BoundAdj {
  double d_phi = 0, d_beta = 0;
  Mat d_psi_y, d_phi_big, d_kmm;
};

static BoundAdj adjoints_from_core(const Core& c, const Stats& st, double beta, Index n, Index d) {
  const double dd = double(d);
  BoundAdj adj;
  adj.d_phi = -0.5 * beta * dd;
  adj.d_psi_y = c.g;
  for (double& x : adj.d_psi_y.v) x *= beta * beta;
  Mat ggt = matmul(c.g, transpose(c.g));
  symmetrize(ggt);
  const Index m = c.a.r;
  adj.d_phi_big = Mat(m, m);
  for (size_t i = 0; i < ggt.v.size(); ++i)
    adj.d_phi_big.v[i] = -0.5 * beta * dd * c.a_inv.v[i] - 0.5 * beta * beta * beta * ggt.v[i] +
                         0.5 * beta * dd * c.kmm_inv.v[i];
  Mat kpk = matmul(matmul(c.kmm_inv, st.phi_big), c.kmm_inv);
  symmetrize(kpk);
  adj.d_kmm = Mat(m, m);
  for (size_t i = 0; i < ggt.v.size(); ++i)
    adj.d_kmm.v[i] = 0.5 * dd * c.kmm_inv.v[i] - 0.5 * dd * c.a_inv.v[i] - 0.5 * beta * beta * ggt.v[i] -
                     0.5 * beta * dd * kpk.v[i];
  double tr_ainv_phi = 0, tr_psig = 0, tr_gphig = 0, tr_kinv_phi = 0;
  Mat phig = matmul(st.phi_big, c.g);
  for (size_t i = 0; i < c.a_inv.v.size(); ++i) {
    tr_ainv_phi += c.a_inv.v[i] * st.phi_big.v[i];
    tr_kinv_phi += c.kmm_inv.v[i] * st.phi_big.v[i];
  }
  for (size_t i = 0; i < c.g.v.size(); ++i) {
    tr_psig += st.psi_y.v[i] * c.g.v[i];
    tr_gphig += c.g.v[i] * phig.v[i];
  }
  adj.d_beta = 0.5 * dd * double(n) / beta - 0.5 * dd * tr_ainv_phi - 0.5 * st.yy + beta * tr_psig -
               0.5 * beta * beta * tr_gphig - 0.5 * dd * st.phi + 0.5 * dd * tr_kinv_phi;
  return adj;
}

// ---------------------------------------------------------------------------
// Data-parallel engine, parallel.hpp
// ---------------------------------------------------------------------------
static std::vector<std::pair<Index, Index>> make_partition(Index n, int p) {
  require(p >= 1, "make_partition: worker count must be >= 1");
  require(Index(p) <= n, "make_partition: more workers than datapoints");
  std::vector<std::pair<Index, Index>> sh;
  const Index base = n / p, rem = n % p;
  Index at = 0;
  for (int i = 0; i < p; ++i) {
    Index len = base + (Index(i) < rem ? 1 : 0);
    sh.emplace_back(at, at + len);
    at += len;
  }
  return sh;
}

struct AdjRequest {
  Adj stats;
  const Mat *a_inv = nullptr, *g = nullptr, *kmm_inv = nullptr;
  double beta = 1.0;
  Index d_out = 0;
};

struct Report {
  Stats stats;
  double kl = 0.0;
  bool has_grads = false;
  Mat d_mu, d_s, d_z;
  double d_variance = 0.0, d_beta = 0.0;
  std::vector<double> d_ls;
};

static double beta_share(const Stats& st, const AdjRequest& r) {  // parallel.hpp:185-195
  const double dd = double(r.d_out), beta = r.beta;
  double tr_ainv_phi = 0, tr_psig = 0, tr_gphig = 0, tr_kinv_phi = 0;
  for (size_t i = 0; i < st.phi_big.v.size(); ++i) {
    tr_ainv_phi += r.a_inv->v[i] * st.phi_big.v[i];
    tr_kinv_phi += r.kmm_inv->v[i] * st.phi_big.v[i];
  }
  Mat phig = matmul(st.phi_big, *r.g);
  for (size_t i = 0; i < r.g->v.size(); ++i) {
    tr_psig += st.psi_y.v[i] * r.g->v[i];
    tr_gphig += r.g->v[i] * phig.v[i];
  }
  return 0.5 * dd * double(st.n_count) / beta - 0.5 * dd * tr_ainv_phi - 0.5 * st.yy + beta * tr_psig -
         0.5 * beta * beta * tr_gphig - 0.5 * dd * st.phi + 0.5 * dd * tr_kinv_phi;
}

// Worker::pass, parallel.hpp:132-176
static Report worker_pass(bool latent, const View& x_or_mu, const View& s, const View& y, const View& z,
                          const Kernel& k, const Tiles& t, const AdjRequest* req) {
  Report rep;
  Grads grads;
  if (latent) {
    sweep_stats(true, x_or_mu, s, y, z, k, t, req ? &req->stats : nullptr, rep.stats, req ? &grads : nullptr);
    double kl = 0.0;
    for (Index j = 0; j < s.c; ++j)
      for (Index i = 0; i < s.r; ++i) {
        double sv = s(i, j), mv = x_or_mu(i, j);
        kl += sv + mv * mv - std::log(sv) - 1.0;
      }
    rep.kl = 0.5 * kl;
  } else {
    sweep_stats(false, x_or_mu, View{}, y, z, k, t, req ? &req->stats : nullptr, rep.stats, req ? &grads : nullptr);
  }
  if (req) {
    rep.has_grads = true;
    rep.d_z = std::move(grads.d_z);
    rep.d_variance = grads.d_variance;
    rep.d_ls = std::move(grads.d_ls);
    if (latent) {
      rep.d_mu = std::move(grads.d_mu);
      rep.d_s = std::move(grads.d_s);
      for (Index j = 0; j < s.c; ++j)
        for (Index i = 0; i < s.r; ++i) {
          rep.d_mu(i, j) -= x_or_mu(i, j);
          rep.d_s(i, j) -= 0.5 * (1.0 - 1.0 / s(i, j));
        }
    }
    rep.d_beta = beta_share(rep.stats, *req);
  }
  return rep;
}

struct EvalOut {
  Breakdown bd;
  Stats stats;
  Mat d_mu, d_s, d_z;
  double d_variance = 0, d_beta = 0;
  std::vector<double> d_ls;
  double wall_s = 0, coordinator_s = 0;
};

template <class F>
static std::vector<Report> run_pass(int p, F&& fn) {
  std::vector<Report> reports(p);
  if (p == 1) {
    reports[0] = fn(0);
    return reports;
  }
  std::vector<std::thread> th;
  std::exception_ptr err;
  std::mutex mu;
  for (int i = 0; i < p; ++i)
    th.emplace_back([&, i] {
      try {
        reports[i] = fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
  return reports;
}

static Report reduce(const std::vector<Report>& reps) {  // parallel.hpp:222-258 (ascending shard order)
  Report out;
  out.stats = Stats::zero(reps[0].stats.psi_y.r, reps[0].stats.psi_y.c);
  out.has_grads = reps[0].has_grads;
  if (out.has_grads) {
    out.d_z = Mat(reps[0].d_z.r, reps[0].d_z.c);
    out.d_ls.assign(reps[0].d_ls.size(), 0.0);
  }
  for (const Report& r : reps) {
    out.stats.add(r.stats);
    out.kl += r.kl;
    if (out.has_grads) {
      for (size_t i = 0; i < out.d_z.v.size(); ++i) out.d_z.v[i] += r.d_z.v[i];
      out.d_variance += r.d_variance;
      for (size_t i = 0; i < out.d_ls.size(); ++i) out.d_ls[i] += r.d_ls[i];
      out.d_beta += r.d_beta;
    }
  }
  return out;
}

// Engine::evaluate(with_grads), parallel.hpp:370-450
static EvalOut engine_evaluate(bool latent, const View& x_or_mu, const View& s, const View& y, const View& z,
                               const Kernel& k, double beta, int workers, const Tiles& tiles,
                               double jitter_factor, bool with_grads) {
  using clk = std::chrono::steady_clock;
  tiles.validate();
  const Index n = y.r, d = y.c;
  auto part = make_partition(n, workers);
  const int p = int(part.size());
  auto t0 = clk::now();
  auto shard = [&](int i, const AdjRequest* req) {
    Index b = part[i].first, len = part[i].second - part[i].first;
    return worker_pass(latent, x_or_mu.rows(b, len), latent ? s.rows(b, len) : View{}, y.rows(b, len), z, k, tiles,
                       req);
  };
  std::vector<Report> pass1 = run_pass(p, [&](int i) { return shard(i, nullptr); });
  Report red = reduce(pass1);
  auto tc0 = clk::now();
  GramFactor gram = factor_gram(z, k, jitter_factor);
  Core core = bound_core(red.stats, gram.kmm, beta, n, d);
  EvalOut out;
  out.stats = red.stats;
  out.bd = core.bd;
  if (latent) {
    out.bd.kl = -red.kl;
    out.bd.total = out.bd.sum();
  }
  double coord = 0.0;
  if (with_grads) {
    BoundAdj adj = adjoints_from_core(core, red.stats, beta, n, d);
    AdjRequest req;
    req.stats.d_phi = adj.d_phi;
    req.stats.d_psi_y = view(adj.d_psi_y);
    req.stats.d_phi_big = view(adj.d_phi_big);
    req.a_inv = &core.a_inv;
    req.g = &core.g;
    req.kmm_inv = &core.kmm_inv;
    req.beta = beta;
    req.d_out = d;
    coord += std::chrono::duration<double>(clk::now() - tc0).count();
    std::vector<Report> pass2 = run_pass(p, [&](int i) { return shard(i, &req); });
    Report red2 = reduce(pass2);
    auto tc1 = clk::now();
    KernGrads gg = kern_grads(z, z, k, view(adj.d_kmm));
    out.d_z = red2.d_z;
    for (size_t i = 0; i < out.d_z.v.size(); ++i) out.d_z.v[i] += gg.d_z.v[i] + gg.d_x.v[i];
    double tr = 0.0;
    for (Index i = 0; i < adj.d_kmm.r; ++i) tr += adj.d_kmm(i, i);
    out.d_variance = red2.d_variance + gg.d_variance + gram.jitter_factor * tr;
    out.d_ls = red2.d_ls;
    for (size_t i = 0; i < out.d_ls.size(); ++i) out.d_ls[i] += gg.d_ls[i];
    out.d_beta = red2.d_beta;
    if (latent) {
      const Index q = x_or_mu.c;
      out.d_mu = Mat(n, q);
      out.d_s = Mat(n, q);
      for (int i = 0; i < p; ++i) {
        Index b = part[i].first, len = part[i].second - part[i].first;
        for (Index j = 0; j < q; ++j)
          for (Index r = 0; r < len; ++r) {
            out.d_mu(b + r, j) = pass2[i].d_mu(r, j);
            out.d_s(b + r, j) = pass2[i].d_s(r, j);
          }
      }
    }
    coord += std::chrono::duration<double>(clk::now() - tc1).count();
  } else {
    coord += std::chrono::duration<double>(clk::now() - tc0).count();
  }
  out.coordinator_s = coord;
  out.wall_s = std::chrono::duration<double>(clk::now() - t0).count();
  return out;
}

// ---------------------------------------------------------------------------
// C ABI for the test / baseline harness (ctypes).  Errors: 0 ok, 1 invalid
// argument (std::invalid_argument), 2 numeric (NumericError), 3 other.
// ---------------------------------------------------------------------------

// ---------------------------------------------------------------------------
// The fitting loop: pack / unpack / pack_gradient (optimizer.hpp:20-144), LbfgsState
// (optimizer.hpp:205-458) and FitSession (model.hpp:100-168) over the oracle engine.
// ---------------------------------------------------------------------------
namespace fitref {
using Vec = std::vector<double>;
static double vdot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
static double vnorm(const Vec& a) { return std::sqrt(vdot(a, a)); }

struct Layout {
  Index q, m, n;
  bool latent;
  Index size() const { return 2 + q + m * q + (latent ? 2 * n * q : 0); }
  Index z_off() const { return 2 + q; }
  Index mu_off() const { return z_off() + m * q; }
  Index s_off() const { return mu_off() + n * q; }
};

struct Params {
  double var, beta;
  Vec ls;
  Mat z, mu, s;
};

static Vec pack(const Params& p, const Layout& L) {
  Vec v(size_t(L.size()));
  v[0] = std::log(p.beta);
  v[1] = std::log(p.var);
  for (Index j = 0; j < L.q; ++j) v[size_t(2 + j)] = std::log(p.ls[size_t(j)]);
  for (Index i = 0; i < L.m; ++i)
    for (Index j = 0; j < L.q; ++j) v[size_t(L.z_off() + i * L.q + j)] = p.z(i, j);
  if (L.latent)
    for (Index i = 0; i < L.n; ++i)
      for (Index j = 0; j < L.q; ++j) {
        v[size_t(L.mu_off() + i * L.q + j)] = p.mu(i, j);
        v[size_t(L.s_off() + i * L.q + j)] = std::log(p.s(i, j));
      }
  return v;
}

static Params unpack(const Vec& v, const Layout& L) {
  Params p;
  p.beta = std::exp(v[0]);
  p.var = std::exp(v[1]);
  p.ls.resize(size_t(L.q));
  for (Index j = 0; j < L.q; ++j) p.ls[size_t(j)] = std::exp(v[size_t(2 + j)]);
  p.z = Mat(L.m, L.q);
  for (Index i = 0; i < L.m; ++i)
    for (Index j = 0; j < L.q; ++j) p.z(i, j) = v[size_t(L.z_off() + i * L.q + j)];
  if (L.latent) {
    p.mu = Mat(L.n, L.q);
    p.s = Mat(L.n, L.q);
    for (Index i = 0; i < L.n; ++i)
      for (Index j = 0; j < L.q; ++j) {
        p.mu(i, j) = v[size_t(L.mu_off() + i * L.q + j)];
        p.s(i, j) = std::exp(v[size_t(L.s_off() + i * L.q + j)]);
      }
  }
  return p;
}

struct Lbfgs {
  int memory = 10;
  double c1 = 1e-4, c2 = 0.9, g_tol = 1e-5, f_tol = 1e-9;
  int max_iters = 500, max_evals = 0, max_ls = 40;
  Vec x, g;
  double value = 0.0;
  struct Pair {
    Vec s, y;
    double rho;
  };
  std::deque<Pair> hist;
  int iter = 0, evals = 0;
  bool done = false;
  int status = -1;
  std::function<double(const Vec&, Vec&)> f;

  double eval(const Vec& xx, Vec& gg) {
    ++evals;
    return f(xx, gg);
  }
  bool zoom(const Vec& dir, double f0, double slope0, double alo, double flo, double dlo, double ahi, double fhi,
            double dhi, double& aout, Vec& xout, double& fout, Vec& gout) {
    Vec gg(x.size());
    for (int it = 0; it < max_ls; ++it) {
      if (max_evals > 0 && evals >= max_evals) return false;
      double a = 0.0;
      {
        const double d1 = dlo + dhi - 3.0 * (flo - fhi) / (alo - ahi);
        const double disc = d1 * d1 - dlo * dhi;
        if (disc > 0.0) {
          const double d2 = std::sqrt(disc) * (ahi > alo ? 1.0 : -1.0);
          a = ahi - (ahi - alo) * (dhi + d2 - d1) / (dhi - dlo + 2.0 * d2);
        }
        const double lo = std::min(alo, ahi), hi = std::max(alo, ahi), w = hi - lo;
        if (!(a > lo + 0.05 * w && a < hi - 0.05 * w)) a = 0.5 * (alo + ahi);
      }
      for (size_t i = 0; i < x.size(); ++i) xout[i] = x[i] + a * dir[i];
      const double fa = eval(xout, gg);
      const double dphi = vdot(gg, dir);
      if (!std::isfinite(fa) || fa > f0 + c1 * a * slope0 || fa >= flo) {
        ahi = a;
        fhi = fa;
        dhi = dphi;
      } else {
        if (std::abs(dphi) <= -c2 * slope0) {
          aout = a;
          fout = fa;
          gout = gg;
          return true;
        }
        if (dphi * (ahi - alo) >= 0.0) {
          ahi = alo;
          fhi = flo;
          dhi = dlo;
        }
        alo = a;
        flo = fa;
        dlo = dphi;
      }
      if (std::abs(ahi - alo) < 1e-16 * std::max(1.0, std::abs(alo))) break;
    }
    if (flo < f0 && alo > 0.0) {
      for (size_t i = 0; i < x.size(); ++i) xout[i] = x[i] + alo * dir[i];
      fout = eval(xout, gout);
      aout = alo;
      return std::isfinite(fout) && fout < f0;
    }
    return false;
  }
  bool line_search(const Vec& dir, double slope0, double a0, double& aout, Vec& xout, double& fout, Vec& gout) {
    const double f0 = value;
    double ap = 0.0, fp = f0, dp = slope0, a = a0;
    Vec gg(x.size());
    for (int it = 0; it < max_ls; ++it) {
      if (max_evals > 0 && evals >= max_evals) return false;
      for (size_t i = 0; i < x.size(); ++i) xout[i] = x[i] + a * dir[i];
      const double fa = eval(xout, gg);
      const double dphi = vdot(gg, dir);
      if (!std::isfinite(fa)) {
        a = 0.5 * (ap + a);
        continue;
      }
      if (fa > f0 + c1 * a * slope0 || (it > 0 && fa >= fp))
        return zoom(dir, f0, slope0, ap, fp, dp, a, fa, dphi, aout, xout, fout, gout);
      if (std::abs(dphi) <= -c2 * slope0) {
        aout = a;
        fout = fa;
        gout = gg;
        return true;
      }
      if (dphi >= 0.0) return zoom(dir, f0, slope0, a, fa, dphi, ap, fp, dp, aout, xout, fout, gout);
      ap = a;
      fp = fa;
      dp = dphi;
      a = std::min(2.0 * a, 1e10);
      if (a >= 1e10) return false;
    }
    return false;
  }
  bool step() {
    if (done) return false;
    const double gn = vnorm(g);
    if (gn <= g_tol) {
      done = true;
      status = 0;
      return false;
    }
    if (max_iters >= 0 && iter >= max_iters) {
      done = true;
      status = 2;
      return false;
    }
    Vec dir(g.size());
    for (size_t i = 0; i < g.size(); ++i) dir[i] = -g[i];
    if (!hist.empty()) {
      std::vector<double> al(hist.size());
      for (Index i = Index(hist.size()) - 1; i >= 0; --i) {
        al[size_t(i)] = hist[size_t(i)].rho * vdot(hist[size_t(i)].s, dir);
        for (size_t k = 0; k < dir.size(); ++k) dir[k] -= al[size_t(i)] * hist[size_t(i)].y[k];
      }
      const auto& last = hist.back();
      const double sc = vdot(last.s, last.y) / vdot(last.y, last.y);
      for (double& v : dir) v *= sc;
      for (size_t i = 0; i < hist.size(); ++i) {
        const double b = hist[i].rho * vdot(hist[i].y, dir);
        for (size_t k = 0; k < dir.size(); ++k) dir[k] += (al[i] - b) * hist[i].s[k];
      }
    }
    double slope = vdot(g, dir);
    if (slope >= 0.0) {
      hist.clear();
      for (size_t i = 0; i < g.size(); ++i) dir[i] = -g[i];
      slope = vdot(g, dir);
    }
    const double a0 = hist.empty() ? std::min(1.0, 1.0 / std::max(1.0, gn)) : 1.0;
    Vec xn(x.size()), gnv(x.size());
    double fnew = 0.0, a = 0.0;
    if (!line_search(dir, slope, a0, a, xn, fnew, gnv)) {
      done = true;
      status = (max_evals > 0 && evals >= max_evals) ? 3 : 4;
      return false;
    }
    Vec sv(x.size()), yv(x.size());
    for (size_t i = 0; i < x.size(); ++i) {
      sv[i] = xn[i] - x[i];
      yv[i] = gnv[i] - g[i];
    }
    const double sy = vdot(sv, yv);
    if (sy > 1e-16 * vnorm(sv) * vnorm(yv)) {
      hist.push_back({sv, yv, 1.0 / sy});
      if (int(hist.size()) > memory) hist.pop_front();
    }
    const double fprev = value;
    x = xn;
    value = fnew;
    g = gnv;
    ++iter;
    if (vnorm(g) <= g_tol) {
      done = true;
      status = 0;
    } else if (std::abs(fprev - value) <= f_tol * std::max({std::abs(fprev), std::abs(value), 1.0})) {
      done = true;
      status = 1;
    }
    return true;
  }
};
}  // namespace fitref

static thread_local std::string g_err;

template <class F>
static int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

static View cv(const double* p, Index r, Index c, Index ld) { return View{p, r, c, ld ? ld : r}; }
static void put(const Mat& m, double* out, Index ld) {
  if (!out) return;
  if (!ld) ld = m.r;
  for (Index j = 0; j < m.c; ++j)
    for (Index i = 0; i < m.r; ++i) out[i + j * ld] = m(i, j);
}
static Kernel mk_kernel(double var, const double* ls, Index q) {
  Kernel k;
  k.variance = var;
  k.ls.assign(ls, ls + q);
  return k;
}

}  // namespace oracle

using namespace oracle;

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

// Restates detail::sweep_stats; all matrices column-major, ld = rows when 0.
// stats_out layout: [phi, yy, n_count]; psi_y_out M x D; phi_big_out M x M.
int oracle_sweep_stats(int expected, int64_t n, int64_t q, int64_t m, int64_t d, const double* mu, const double* s,
                       const double* y, const double* z, double variance, const double* ls, int64_t block_span,
                       int64_t thread_span, int has_adj, double d_phi, const double* d_psi_y,
                       const double* d_phi_big, double* scalars_out, double* psi_y_out, double* phi_big_out,
                       double* d_mu_out, double* d_s_out, double* d_z_out, double* d_var_out, double* d_ls_out) {
  return guard([&] {
    Kernel k = mk_kernel(variance, ls, q);
    Tiles t{block_span, thread_span};
    Adj adj{d_phi, cv(d_psi_y, m, d, 0), cv(d_phi_big, m, m, 0)};
    Stats st;
    Grads g;
    sweep_stats(expected != 0, cv(mu, n, q, 0), expected ? cv(s, n, q, 0) : View{}, cv(y, n, d, 0), cv(z, m, q, 0),
                k, t, has_adj ? &adj : nullptr, st, d_z_out ? &g : nullptr);
    scalars_out[0] = st.phi;
    scalars_out[1] = st.yy;
    scalars_out[2] = double(st.n_count);
    put(st.psi_y, psi_y_out, 0);
    put(st.phi_big, phi_big_out, 0);
    if (d_z_out) {
      if (expected) {
        put(g.d_mu, d_mu_out, 0);
        put(g.d_s, d_s_out, 0);
      }
      put(g.d_z, d_z_out, 0);
      *d_var_out = g.d_variance;
      for (Index j = 0; j < q; ++j) d_ls_out[j] = g.d_ls[j];
    }
  });
}

int oracle_psi1_expected(int64_t n, int64_t q, int64_t m, const double* mu, const double* s, const double* z,
                         double variance, const double* ls, double* out) {
  return guard([&] {
    Mat r = psi1_expected(cv(mu, n, q, 0), cv(s, n, q, 0), cv(z, m, q, 0), mk_kernel(variance, ls, q));
    put(r, out, 0);
  });
}

int oracle_kern_cross(int64_t n, int64_t m, int64_t q, const double* x, const double* z, double variance,
                      const double* ls, double* out) {
  return guard([&] { put(kern_cross(cv(x, n, q, 0), cv(z, m, q, 0), mk_kernel(variance, ls, q)), out, 0); });
}

int oracle_kern_gram(int64_t m, int64_t q, const double* z, double variance, const double* ls, double jitter,
                     double* out, int* near_dup) {
  return guard([&] {
    bool dup = false;
    put(kern_gram(cv(z, m, q, 0), mk_kernel(variance, ls, q), jitter, &dup), out, 0);
    if (near_dup) *near_dup = dup ? 1 : 0;
  });
}

int oracle_kern_grads(int64_t n, int64_t m, int64_t q, const double* x, const double* z, double variance,
                      const double* ls, const double* upstream, double* d_var, double* d_ls, double* d_z,
                      double* d_x) {
  return guard([&] {
    KernGrads g = kern_grads(cv(x, n, q, 0), cv(z, m, q, 0), mk_kernel(variance, ls, q), cv(upstream, n, m, 0));
    *d_var = g.d_variance;
    for (Index j = 0; j < q; ++j) d_ls[j] = g.d_ls[j];
    put(g.d_z, d_z, 0);
    put(g.d_x, d_x, 0);
  });
}

int oracle_factor_gram(int64_t m, int64_t q, const double* z, double variance, const double* ls,
                       double jitter_factor, double* kmm_out, double* jitter_out, double* jf_out,
                       double* log_det_out) {
  return guard([&] {
    GramFactor f = factor_gram(cv(z, m, q, 0), mk_kernel(variance, ls, q), jitter_factor);
    put(f.kmm, kmm_out, 0);
    *jitter_out = f.jitter;
    *jf_out = f.jitter_factor;
    *log_det_out = f.log_det;
  });
}

// bound_core + adjoints_from_core on given statistics. bd_out[7] = total, log_det, data_fit,
// quadratic, trace_phi, trace_kmm, kl.  adj: d_phi, d_beta scalars; d_psi_y M x D; d_phi_big, d_kmm M x M.
int oracle_bound(int64_t m, int64_t d, int64_t n, double phi, double yy, const double* psi_y, const double* phi_big,
                 const double* kmm, double beta, double* bd_out, double* adj_scalars, double* d_psi_y,
                 double* d_phi_big, double* d_kmm) {
  return guard([&] {
    Stats st = Stats::zero(m, d);
    st.phi = phi;
    st.yy = yy;
    st.n_count = n;
    std::copy(psi_y, psi_y + m * d, st.psi_y.v.begin());
    std::copy(phi_big, phi_big + m * m, st.phi_big.v.begin());
    Mat K(m, m);
    std::copy(kmm, kmm + m * m, K.v.begin());
    Core c = bound_core(st, K, beta, n, d);
    const Breakdown& b = c.bd;
    double vals[7] = {b.total, b.log_det, b.data_fit, b.quadratic, b.trace_phi, b.trace_kmm, b.kl};
    std::copy(vals, vals + 7, bd_out);
    if (adj_scalars) {
      BoundAdj a = adjoints_from_core(c, st, beta, n, d);
      adj_scalars[0] = a.d_phi;
      adj_scalars[1] = a.d_beta;
      put(a.d_psi_y, d_psi_y, 0);
      put(a.d_phi_big, d_phi_big, 0);
      put(a.d_kmm, d_kmm, 0);
    }
  });
}

// Engine(kind).evaluate(with_grads).  kind: 0 regression (s ignored), 1 latent.
// bd_out[7]; stats_scalars[3] = phi, yy, n; psi_y M x D; phi_big M x M; grads: d_mu, d_s (N x Q, latent),
// d_z M x Q, gscalars[2] = d_variance, d_beta; d_ls Q; times[2] = wall_s, coordinator_s.
int oracle_engine_evaluate(int kind, int64_t n, int64_t q, int64_t d, int64_t m, const double* x_or_mu,
                           const double* s, const double* y, const double* z, double variance, const double* ls,
                           double beta, int workers, int64_t block_span, int64_t thread_span, double jitter_factor,
                           int with_grads, double* bd_out, double* stats_scalars, double* psi_y, double* phi_big,
                           double* d_mu, double* d_s, double* d_z, double* gscalars, double* d_ls, double* times) {
  return guard([&] {
    Kernel k = mk_kernel(variance, ls, q);
    Tiles t{block_span, thread_span};
    EvalOut o = engine_evaluate(kind == 1, cv(x_or_mu, n, q, 0), kind == 1 ? cv(s, n, q, 0) : View{},
                                cv(y, n, d, 0), cv(z, m, q, 0), k, beta, workers, t, jitter_factor, with_grads != 0);
    const Breakdown& b = o.bd;
    double vals[7] = {b.total, b.log_det, b.data_fit, b.quadratic, b.trace_phi, b.trace_kmm, b.kl};
    std::copy(vals, vals + 7, bd_out);
    stats_scalars[0] = o.stats.phi;
    stats_scalars[1] = o.stats.yy;
    stats_scalars[2] = double(o.stats.n_count);
    put(o.stats.psi_y, psi_y, 0);
    put(o.stats.phi_big, phi_big, 0);
    if (with_grads) {
      if (kind == 1) {
        put(o.d_mu, d_mu, 0);
        put(o.d_s, d_s, 0);
      }
      put(o.d_z, d_z, 0);
      gscalars[0] = o.d_variance;
      gscalars[1] = o.d_beta;
      for (Index j = 0; j < q; ++j) d_ls[j] = o.d_ls[j];
    }
    if (times) {
      times[0] = o.wall_s;
      times[1] = o.coordinator_s;
    }
  });
}

// FitSession over the oracle engine: `iters` sync_steps; values[0..] = -bound per accepted iterate,
// final parameters out (var, ls, beta, z, mu, s).  Returns the L-BFGS status in *status.
int oracle_fit(int kind, int64_t n, int64_t q, int64_t d, int64_t m, const double* x_or_mu, const double* s0,
               const double* y, const double* z0, double variance, const double* ls0, double beta, int workers,
               int iters, double* values, double* grad_norms, int* status, int* evals, double* var_out,
               double* ls_out, double* beta_out, double* z_out, double* mu_out, double* s_out) {
  return guard([&] {
    const bool latent = kind == 1;
    fitref::Layout L{q, m, latent ? n : 0, latent};
    fitref::Params p;
    p.var = variance;
    p.beta = beta;
    p.ls.assign(ls0, ls0 + q);
    p.z = Mat(m, q);
    std::copy(z0, z0 + m * q, p.z.v.begin());
    if (latent) {
      p.mu = Mat(n, q);
      p.s = Mat(n, q);
      std::copy(x_or_mu, x_or_mu + n * q, p.mu.v.begin());
      std::copy(s0, s0 + n * q, p.s.v.begin());
    }
    const View yv = cv(y, n, d, 0);
    fitref::Lbfgs opt;
    opt.f = [&](const fitref::Vec& v, fitref::Vec& g) {  // DistributedObjective (model.hpp:66-84)
      fitref::Params pp = fitref::unpack(v, L);
      Kernel k = mk_kernel(pp.var, pp.ls.data(), q);
      EvalOut r = latent ? engine_evaluate(true, view(pp.mu), view(pp.s), yv, view(pp.z), k, pp.beta, workers,
                                           Tiles{64, 1024}, 1e-6, true)
                         : engine_evaluate(false, cv(x_or_mu, n, q, 0), View{}, yv, view(pp.z), k, pp.beta, workers,
                                           Tiles{64, 1024}, 1e-6, true);
      g.assign(size_t(L.size()), 0.0);  // -pack_gradient (optimizer.hpp:126-144)
      g[0] = -pp.beta * r.d_beta;
      g[1] = -pp.var * r.d_variance;
      for (Index j = 0; j < q; ++j) g[size_t(2 + j)] = -pp.ls[size_t(j)] * r.d_ls[size_t(j)];
      for (Index i = 0; i < m; ++i)
        for (Index j = 0; j < q; ++j) g[size_t(L.z_off() + i * q + j)] = -r.d_z(i, j);
      if (latent)
        for (Index i = 0; i < n; ++i)
          for (Index j = 0; j < q; ++j) {
            g[size_t(L.mu_off() + i * q + j)] = -r.d_mu(i, j);
            g[size_t(L.s_off() + i * q + j)] = -pp.s(i, j) * r.d_s(i, j);
          }
      return -r.bd.total;
    };
    opt.x = fitref::pack(p, L);
    opt.value = opt.eval(opt.x, opt.g);  // initialize
    values[0] = opt.value;
    grad_norms[0] = fitref::vnorm(opt.g);
    int k = 0;
    for (; k < iters && opt.step(); ++k) {
      values[k + 1] = opt.value;
      grad_norms[k + 1] = fitref::vnorm(opt.g);
    }
    *status = opt.done ? opt.status : -1;
    *evals = opt.evals;
    fitref::Params out = fitref::unpack(opt.x, L);
    *var_out = out.var;
    *beta_out = out.beta;
    std::copy(out.ls.begin(), out.ls.end(), ls_out);
    std::copy(out.z.v.begin(), out.z.v.end(), z_out);
    if (latent) {
      std::copy(out.mu.v.begin(), out.mu.v.end(), mu_out);
      std::copy(out.s.v.begin(), out.s.v.end(), s_out);
    }
  });
}

// Prediction (model.hpp:181-217): finalize() = stats at the current parameters, factor_gram, bound_core
// (model.hpp:265-276, 353-364), then predict_from_cache on kern_cross(X*, Z).  obs != 0 adds 1/beta.
int oracle_predict(int kind, int64_t n, int64_t q, int64_t d, int64_t m, const double* x_or_mu, const double* s,
                   const double* y, const double* z, double variance, const double* ls, double beta,
                   double jitter_factor, int64_t t, const double* x_star, int obs, double* mean_out,
                   double* var_out, double* bound_out) {
  return guard([&] {
    Kernel k = mk_kernel(variance, ls, q);
    const bool latent = kind == 1;
    Stats st;
    sweep_stats(latent, cv(x_or_mu, n, q, 0), latent ? cv(s, n, q, 0) : View{}, cv(y, n, d, 0), cv(z, m, q, 0), k,
                Tiles{64, 1024}, nullptr, st, nullptr);
    GramFactor gram = factor_gram(cv(z, m, q, 0), k, jitter_factor);
    Core core = bound_core(st, gram.kmm, beta, n, d);
    double kl = 0.0;
    if (latent)  // kl_gaussian (bound.hpp:164-169)
      for (Index j = 0; j < q; ++j)
        for (Index i = 0; i < n; ++i) {
          const double mu = x_or_mu[i + j * n], sv = s[i + j * n];
          kl += 0.5 * (sv + mu * mu - std::log(sv) - 1.0);
        }
    *bound_out = core.bd.total - kl;
    Mat ks = kern_cross(cv(x_star, t, q, 0), cv(z, m, q, 0), k);  // T x M
    Mat mean = matmul(ks, core.g);
    for (double& v : mean.v) v *= beta;
    put(mean, mean_out, 0);
    for (Index r = 0; r < t; ++r) {
      double n1 = 0.0, n2 = 0.0;  // |L_k^-1 k*|^2, |L_a^-1 k*|^2 by forward substitution
      for (int which = 0; which < 2; ++which) {
        const Mat& L = which == 0 ? gram.L : core.La;
        std::vector<double> x(static_cast<size_t>(m));
        double acc = 0.0;
        for (Index i = 0; i < m; ++i) {
          double sum = ks(r, i);
          for (Index kk = 0; kk < i; ++kk) sum -= L(i, kk) * x[size_t(kk)];
          x[size_t(i)] = sum / L(i, i);
          acc += x[size_t(i)] * x[size_t(i)];
        }
        (which == 0 ? n1 : n2) = acc;
      }
      double v = std::max(variance - n1 + n2, 1e-15 * variance);
      if (obs) v += 1.0 / beta;
      for (Index c = 0; c < d; ++c) var_out[r + c * t] = v;
    }
  });
}

// Rng restatement: fills column-major rows x cols with next_normal() in row-major visiting order
// (common.hpp:86-91).  Returns the generator state so callers can chain.
void oracle_rng_normal_matrix(uint64_t seed, int64_t rows, int64_t cols, double* out) {
  Rng r(seed);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) out[i + j * rows] = r.normal();
}

// init_gplvm's Z rows (model.hpp:420-429): partial Fisher-Yates over 0..n-1 with Rng(seed).
void oracle_rng_choose_rows(uint64_t seed, int64_t n, int64_t m, int64_t* out) {
  Rng r(seed);
  std::vector<int64_t> idx(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) idx[size_t(i)] = i;
  for (int64_t i = 0; i < m; ++i) {
    const int64_t j = i + int64_t(r.index(uint64_t(n - i)));
    std::swap(idx[size_t(i)], idx[size_t(j)]);
    out[i] = idx[size_t(i)];
  }
}

void oracle_rng_uniform(uint64_t seed, int64_t count, double* out) {
  Rng r(seed);
  for (Index i = 0; i < count; ++i) out[i] = r.uniform();
}

int oracle_make_partition(int64_t n, int p, int64_t* begins, int64_t* ends) {
  return guard([&] {
    auto sh = make_partition(n, p);
    for (int i = 0; i < p; ++i) {
      begins[i] = sh[i].first;
      ends[i] = sh[i].second;
    }
  });
}

}  // extern "C"
