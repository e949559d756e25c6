// Compiles include/sgp_b200_shim.hpp against a minimal Eigen-shaped column-major matrix (the
// reference's types need Eigen, absent here) and runs the reference's SPEC KATs through it:
// psi2 of N=M=Q=1, mu=0, S=1, z=0 -> 1/sqrt(3); stats N=1 -> all ones.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "sgp_b200_shim.hpp"

struct Matrix {
  long r = 0, c = 0;
  std::vector<double> v;
  Matrix() = default;
  Matrix(long rr, long cc) : r(rr), c(cc), v(rr * cc, 0.0) {}
  static Matrix Zero(long rr, long cc) { return Matrix(rr, cc); }
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  long rows() const { return r; }
  long cols() const { return c; }
  long outerStride() const { return r; }
  double& operator()(long i, long j) { return v[i + j * r]; }
};
struct Vector {
  std::vector<double> v;
  void setZero(long n) { v.assign(n, 0.0); }
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  long size() const { return (long)v.size(); }
};
struct KernelSpec { double variance = 1.0; Vector lengthscales; };
struct TileConfig { long block_span = 64, thread_span = 1024; };
struct SufficientStats { double phi = 0; Matrix psi_y, phi_big; double yy = 0; long n_count = 0; };
struct StatsAdjoints { double d_phi = 0; Matrix d_psi_y, d_phi_big; };
struct StatsGrads { Matrix d_mu, d_s, d_z; double d_variance = 0; Vector d_lengthscales; };
struct NumericError : std::runtime_error { using std::runtime_error::runtime_error; };

int main() {
  Matrix mu(1, 1), s(1, 1), y(1, 1), z(1, 1);
  s(0, 0) = 1.0;
  y(0, 0) = 1.0;
  KernelSpec k;
  k.lengthscales.v = {1.0};
  SufficientStats st;
  try {
    sgp_b200::sweep_stats<NumericError, Matrix>(true, mu, s, y, z, k, TileConfig{}, (StatsAdjoints*)nullptr, st,
                                                (StatsGrads*)nullptr);
  } catch (const std::runtime_error& e) {
    std::printf("NODEVICE %s\n", e.what());
    return 3;
  }
  const double want = 1.0 / std::sqrt(3.0);
  std::printf("psi2 %.17g want %.17g phi %.17g n %ld\n", st.phi_big(0, 0), want, st.phi, st.n_count);
  SufficientStats sd;
  sgp_b200::sweep_stats<NumericError, Matrix>(false, mu, Matrix(), y, z, k, TileConfig{}, (StatsAdjoints*)nullptr,
                                              sd, (StatsGrads*)nullptr);
  std::printf("det %.17g %.17g %.17g %.17g\n", sd.phi, sd.psi_y(0, 0), sd.phi_big(0, 0), sd.yy);
  const bool ok = std::fabs(st.phi_big(0, 0) - want) < 1e-6 && st.phi == 1.0 && std::fabs(sd.psi_y(0, 0) - 1) < 1e-6 &&
                  std::fabs(sd.phi_big(0, 0) - 1) < 1e-6 && sd.yy == 1.0;
  return ok ? 0 : 1;
}
