// sgp_b200_shim.hpp -- reference-side binding of libsgpx (include/sgpx.h).
//
// A maintainer of the reference adds this header next to proj/include/sgp/psi_stats.hpp and
// routes detail::sweep_stats (psi_stats.hpp:108-326) through it; every caller above
// (stats_* wrappers :332-426, Worker::pass parallel.hpp:146,151, finalize model.hpp:273,359)
// stays unchanged.  Templated on the matrix type so it binds Eigen::Ref<const MatrixXd> in the
// reference and any column-major type with data()/rows()/cols()/outerStride() elsewhere.
//
// Errors are rethrown as the reference's types: SGPX_INVALID_ARGUMENT -> std::invalid_argument
// (common.hpp:24-26), SGPX_NUMERIC -> NumericErrorT (sgp::NumericError, common.hpp:20-22).
#pragma once
#include <stdexcept>
#include <string>
#include <vector>

#include "sgpx.h"

namespace sgp_b200 {

template <class M>
inline sgpx_cmat cview(const M& m) {
  return sgpx_cmat{m.rows() * m.cols() ? m.data() : nullptr, (int64_t)m.rows(), (int64_t)m.cols(),
                   (int64_t)(m.cols() > 1 ? m.outerStride() : m.rows())};
}
template <class M>
inline sgpx_mmat mview(M& m) {
  return sgpx_mmat{m.rows() * m.cols() ? m.data() : nullptr, (int64_t)m.rows(), (int64_t)m.cols(),
                   (int64_t)(m.cols() > 1 ? m.outerStride() : m.rows())};
}

template <class NumericErrorT>
inline void check(int rc) {
  if (rc == SGPX_OK) return;
  const std::string msg = sgpx_last_error();
  if (rc == SGPX_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == SGPX_NUMERIC) throw NumericErrorT(msg);
  throw std::runtime_error("libsgpx: " + msg);
}

// One context per host thread (the reference calls sweep_stats concurrently from run_pass threads).
inline sgpx_ctx* thread_context(int device = 0) {
  struct Holder {
    sgpx_ctx* c = nullptr;
    ~Holder() {
      if (c) sgpx_ctx_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.c && sgpx_ctx_create(device, &h.c) != SGPX_OK) {
    h.c = nullptr;
    throw std::runtime_error(std::string("libsgpx: ") + sgpx_last_error());
  }
  return h.c;
}

// Drop-in body for sgp::detail::sweep_stats.  Matrix/Vector: the reference's Eigen types;
// Stats/Adjoints/Grads: SufficientStats / StatsAdjoints / StatsGrads (psi_stats.hpp:31-71);
// Kernel: KernelSpec (kernels.hpp:13-33); Tiles: TileConfig (common.hpp:30-37).
template <class NumericErrorT, class Matrix, class MuT, class ST, class YT, class ZT, class Kernel, class Tiles,
          class Adjoints, class Stats, class Grads>
void sweep_stats(bool expected, const MuT& mu, const ST& s, const YT& y, const ZT& z, const Kernel& kernel,
                 const Tiles& tiles, const Adjoints* adj, Stats& stats, Grads* grads) {
  const auto m = z.rows(), d = y.cols(), n = mu.rows(), q = mu.cols();
  std::vector<double> ls(kernel.lengthscales.data(), kernel.lengthscales.data() + kernel.lengthscales.size());
  sgpx_kernel_spec ks{kernel.variance, ls.data(), (int64_t)ls.size()};
  sgpx_tile_config tc{(int64_t)tiles.block_span, (int64_t)tiles.thread_span};
  stats.psi_y = Matrix::Zero(m, d);
  stats.phi_big = Matrix::Zero(m, m);
  sgpx_sufficient_stats cs{0.0, mview(stats.psi_y), mview(stats.phi_big), 0.0, 0};
  sgpx_stats_adjoints ca{};
  if (adj) ca = sgpx_stats_adjoints{adj->d_phi, cview(adj->d_psi_y), cview(adj->d_phi_big)};
  sgpx_stats_grads cg{};
  if (grads) {
    grads->d_mu = expected ? Matrix(Matrix::Zero(n, q)) : Matrix();
    grads->d_s = expected ? Matrix(Matrix::Zero(n, q)) : Matrix();
    grads->d_z = Matrix::Zero(m, q);
    grads->d_lengthscales.setZero(q);
    cg = sgpx_stats_grads{mview(grads->d_mu), mview(grads->d_s), mview(grads->d_z), 0.0,
                          grads->d_lengthscales.data()};
  }
  check<NumericErrorT>(sgpx_sweep_stats(thread_context(), expected ? 1 : 0, cview(mu), cview(s), cview(y), cview(z),
                                        &ks, &tc, adj ? &ca : nullptr, &cs, grads ? &cg : nullptr));
  stats.phi = cs.phi;
  stats.yy = cs.yy;
  stats.n_count = cs.n_count;
  if (grads) grads->d_variance = cg.d_variance;
}

}  // namespace sgp_b200
