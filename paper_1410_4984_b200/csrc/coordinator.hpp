// coordinator.hpp -- the indistributable M-sized algebra of one bound+gradient
// evaluation, fp64 on the host, run redundantly on every rank after the
// statistics allreduce (so no broadcast is needed).
//
// Reference: kern_gram / kern_grads / factor_gram (proj/include/sgp/kernels.hpp:83-197),
// factor_spd / bound_core / adjoints_from_core (proj/include/sgp/bound.hpp:52-226),
// and the coordinator block of Engine::evaluate (proj/include/sgp/parallel.hpp:378-421).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace sgpx {

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// File input / output failures (the reference's std::runtime_error in io.hpp).
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
inline void require(bool c, const std::string& msg) {
  if (!c) throw InvalidArgument(msg);
}

namespace coord {

// Dense column-major fp64 matrix.
struct Mat {
  int64_t r = 0, c = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(int64_t rows, int64_t cols) : r(rows), c(cols), v(size_t(rows * cols), 0.0) {}
  double& operator()(int64_t i, int64_t j) { return v[size_t(i + j * r)]; }
  double operator()(int64_t i, int64_t j) const { return v[size_t(i + j * r)]; }
  double* col(int64_t j) { return v.data() + j * r; }
  const double* col(int64_t j) const { return v.data() + j * r; }
};

struct Kernel {
  double variance = 1.0;
  std::vector<double> ls;
  int64_t q() const { return int64_t(ls.size()); }
  void validate() const;
};

// Lower Cholesky; false on a non-positive (or NaN) pivot, like Eigen::LLT.
bool cholesky(const Mat& a, Mat& L);
double log_det_chol(const Mat& L);
// Solve (L L^T) X = B in place.
void chol_solve(const Mat& L, Mat& B);
// Symmetric (L L^T)^{-1}, symmetrised as 0.5 (X + X^T) like bound.hpp:98-101.
Mat chol_inverse(const Mat& L);
// C = op(A) * op(B).
Mat gemm(const Mat& A, bool ta, const Mat& B, bool tb);

Mat kern_gram(const Mat& z, const Kernel& k, double jitter, bool* near_dup);

struct GramFactor {
  Mat kmm, L;
  double jitter = 0.0, jitter_factor = 0.0, log_det = 0.0;
};
GramFactor factor_gram(const Mat& z, const Kernel& k, double jitter_factor);

struct Breakdown {
  double total = 0, log_det = 0, data_fit = 0, quadratic = 0, trace_phi = 0, trace_kmm = 0, kl = 0;
  double sum() const { return log_det + data_fit + quadratic + trace_phi + trace_kmm + kl; }
};

struct Stats {
  double phi = 0, yy = 0, n = 0, kl = 0;
  Mat psi_y, phi_big;
};

// Unpack the allreduce #1 payload (layout: sgpx.h sgpx_packed_stats_count).
Stats unpack_stats(const double* packed, int64_t m, int64_t d);

struct Adjoints {
  double d_phi = 0, d_beta = 0;
  Mat d_psi_y, d_phi_big, d_kmm;
};

struct Result {
  Breakdown bd;
  GramFactor gram;
  Adjoints adj;
  // deferred adjoints: d_kmm and d_beta are only needed by the host-side gradient assembly, so
  // the engine computes them (complete_adjoints) while the gradient kernels run
  bool deferred = false;
  Mat kmm_inv, a_inv, g, ggt;
  double ap = 0, kp = 0, pg = 0;
};

// factor_gram + bound_core (+ KL for the latent model) + adjoints_from_core.  With
// defer_host_only, only the adjoints the device pass needs (d_phi, d_psi_y, d_phi_big) are formed;
// complete_adjoints adds d_kmm and d_beta (same arithmetic, bitwise identical results).
// The Z-only part of the coordinator (factor_gram and (Kmm)^-1): the engine forms it while the
// statistics pass runs on the device.
struct Prefactor {
  GramFactor gram;
  Mat kmm_inv;
};
Prefactor prefactor(const Mat& z, const Kernel& k, double jitter_factor);

Result coordinate(bool latent, int64_t n, int64_t d, const Stats& st, const Mat& z, const Kernel& k, double beta,
                  double jitter_factor, bool with_adjoints, bool defer_host_only = false,
                  const Prefactor* pre = nullptr);
void complete_adjoints(Result& r, const Stats& st, int64_t n, int64_t d, double beta);

struct KernGrads {
  double d_variance = 0;
  std::vector<double> d_ls;
  Mat d_z;  // d_z + d_x of kern_grads(Z, Z, .)
};
// kern_grads(Z, Z, k, upstream) with the Z- and X-slot gradients summed (parallel.hpp:416-419).
KernGrads kern_grads_zz(const Mat& z, const Kernel& k, const Mat& upstream);

}  // namespace coord
}  // namespace sgpx
