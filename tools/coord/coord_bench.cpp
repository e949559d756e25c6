// coord_bench.cpp -- host timing of the M-sized coordinator (coordinator.cpp) at the C3 shape
// (M = 100, D = 50, Q = 10), with a per-stage breakdown.
//   g++ -std=c++17 -O3 -march=x86-64-v3 -I../../paper_1410_4984_b200/csrc coord_bench.cpp \
//       ../../paper_1410_4984_b200/csrc/coordinator.cpp -o coord_bench
#include <chrono>
#include <cstdio>
#include <random>

#include "coordinator.hpp"

using namespace sgpx::coord;

int main() {
  const int64_t m = 100, d = 50, q = 10, n = 1000000;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  Mat z(m, q);
  for (auto& x : z.v) x = nd(rng);
  Kernel k;
  k.variance = 1.0;
  k.ls.assign(q, 1.0);
  // stats of a plausible shard: Phi = sum of n rank-one terms ~ (n / m) * PD matrix
  Mat b(m, m);
  for (auto& x : b.v) x = nd(rng) * 0.1;
  Stats st;
  st.n = double(n);
  st.phi = double(n);
  st.yy = double(n) * d;
  st.kl = 1000.0;
  st.phi_big = gemm(b, false, b, true);
  for (int64_t i = 0; i < m; ++i) st.phi_big(i, i) += 1.0;
  for (auto& x : st.phi_big.v) x *= double(n) / m;
  st.psi_y = Mat(m, d);
  for (auto& x : st.psi_y.v) x = nd(rng) * 100.0;
  Result r;
  for (int w = 0; w < 3; ++w) r = coordinate(true, n, d, st, z, k, 100.0, 1e-6, true);
  const int reps = 200;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) r = coordinate(true, n, d, st, z, k, 100.0, 1e-6, true);
  auto t1 = std::chrono::steady_clock::now();
  printf("coordinate(with adjoints): %.3f ms  (bound %.6e)\n",
         std::chrono::duration<double, std::milli>(t1 - t0).count() / reps, r.bd.total);
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) r = coordinate(true, n, d, st, z, k, 100.0, 1e-6, false);
  t1 = std::chrono::steady_clock::now();
  printf("coordinate(bound only):    %.3f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count() / reps);
  Mat dummy;
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) dummy = gemm(st.phi_big, false, st.phi_big, false);
  t1 = std::chrono::steady_clock::now();
  printf("gemm 100^3:                %.3f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count() / reps);
  Mat L;
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) cholesky(st.phi_big, L);
  t1 = std::chrono::steady_clock::now();
  printf("cholesky 100:              %.3f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count() / reps);
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) dummy = chol_inverse(L);
  t1 = std::chrono::steady_clock::now();
  printf("chol_inverse 100:          %.3f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count() / reps);
  Mat up(m, m);
  for (auto& x : up.v) x = nd(rng);
  KernGrads kg;
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) kg = kern_grads_zz(z, k, up);
  t1 = std::chrono::steady_clock::now();
  printf("kern_grads_zz:             %.3f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count() / reps);
  return 0;
}
