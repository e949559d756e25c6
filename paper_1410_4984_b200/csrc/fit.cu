// fit.cu -- the optimisation loop around the engine, resident on the device.
//
// Reference: ParameterLayout / pack / unpack / pack_gradient (optimizer.hpp:20-144), LbfgsState
// (optimizer.hpp:205-458: two-loop recursion, strong-Wolfe line search with cubic zoom),
// DistributedObjective (model.hpp:61-92) and FitSession::sync_step (model.hpp:100-168).
//
// The parameter vector, the gradient and the L-BFGS history live in HBM; the objective broadcasts the
// device-resident mu / S to the engine (no host copy of the N x Q segments) and reads the engine's
// d mu / d S in place.  Only the M-sized segment (beta, variance, lengthscales, Z) crosses to the host
// per evaluation, plus the scalars of the dot products the line search branches on.  Every dot
// product is a fixed-order two-level reduction, so a fit is bitwise reproducible.
//
// Internal layout: [log beta, log variance, log l (Q), Z (M x Q row-major), mu (N x Q column-major),
// log S (N x Q column-major)].  The reference packs mu / log S row-major; L-BFGS only uses dot products,
// norms and axpys, which a fixed permutation of the coordinates leaves unchanged, and sgpx_fit_params
// returns the matrices in their natural shapes.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <deque>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sgpx.h"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;
namespace {

constexpr int kDotBlocks = 296;

__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                   double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    s += a[i] * b[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void dot_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// y = a x + b y
__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}

// out = x + a d
__global__ void xpad_kernel(int64_t n, const double* __restrict__ x, double a, const double* __restrict__ d,
                            double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = x[i] + a * d[i];
}

__global__ void exp_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = exp(x[i]);
}

// gradient of -bound in the packed coordinates (pack_gradient, optimizer.hpp:126-144):
// d/d mu = -d mu, d/d log s = -s d s
__global__ void local_grad_kernel(int64_t nq, const double* __restrict__ dmu, const double* __restrict__ ds,
                                  const double* __restrict__ s, double* __restrict__ g_mu, double* __restrict__ g_s) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nq; i += int64_t(gridDim.x) * blockDim.x) {
    g_mu[i] = -dmu[i];
    g_s[i] = -s[i] * ds[i];
  }
}

struct FitError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline unsigned grid_for(int64_t n) { return unsigned(std::min<int64_t>((n + 255) / 256, 148 * 8)); }

}  // namespace
}  // namespace sgpx

using namespace sgpx;

struct sgpx_fit {
  sgpx_engine* eng = nullptr;
  sgpx_ctx* ctx = nullptr;
  cudaStream_t st = nullptr;
  int64_t q = 0, m = 0, n = 0, d = 0;
  bool latent = false;
  int64_t dim = 0, off_z = 0, off_mu = 0, off_s = 0;
  sgpx_lbfgs_options o{};
  // device vectors
  double *x = nullptr, *g = nullptr, *dir = nullptr, *xn = nullptr, *gn = nullptr, *gt = nullptr, *sdev = nullptr;
  double *part = nullptr, *scal = nullptr;
  std::vector<double*> hs, hy;  // history slots
  struct Pair {
    int slot;
    double rho;
  };
  std::deque<Pair> hist;
  std::vector<int> free_slots;
  double* h_scal = nullptr;  // pinned: one dot result
  std::vector<double> h_glob;
  // state
  double value = 0.0;
  int iter = 0, evals = 0, last_step_evals = 0;
  bool done = false;
  int status = -1;
  std::string message;
  std::string err;
  ~sgpx_fit() {
    for (double* p : {x, g, dir, xn, gn, gt, sdev, part, scal})
      if (p) cudaFree(p);
    for (double* p : hs) cudaFree(p);
    for (double* p : hy) cudaFree(p);
    if (h_scal) cudaFreeHost(h_scal);
  }
};

namespace {

void cuok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw FitError(std::string(what) + ": " + cudaGetErrorString(e));
}

void api(int rc) {
  if (rc != SGPX_OK) throw FitError(sgpx_last_error());
}

double dot(sgpx_fit* f, const double* a, const double* b) {
  dot_partial_kernel<<<kDotBlocks, 256, 0, f->st>>>(a, b, f->dim, f->part);
  dot_final_kernel<<<1, 256, 0, f->st>>>(f->part, kDotBlocks, f->scal);
  g_tc_launches.fetch_add(2);
  cuok(cudaMemcpyAsync(f->h_scal, f->scal, sizeof(double), cudaMemcpyDeviceToHost, f->st), "dot");
  cuok(cudaStreamSynchronize(f->st), "dot");
  return *f->h_scal;
}

void axpby(sgpx_fit* f, double a, const double* x, double b, double* y) {
  axpby_kernel<<<grid_for(f->dim), 256, 0, f->st>>>(f->dim, a, x, b, y);
  g_tc_launches.fetch_add(1);
}

void xpad(sgpx_fit* f, const double* x, double a, const double* d, double* out) {
  xpad_kernel<<<grid_for(f->dim), 256, 0, f->st>>>(f->dim, x, a, d, out);
  g_tc_launches.fetch_add(1);
}

void copy(sgpx_fit* f, double* dst, const double* src) {
  cuok(cudaMemcpyAsync(dst, src, sizeof(double) * f->dim, cudaMemcpyDeviceToDevice, f->st), "copy");
}

// The objective of DistributedObjective (model.hpp:66-84): broadcast the unpacked parameters, one
// evaluation with gradients, value = -bound, gradient = -pack_gradient.  NumericError is rethrown
// with the iteration number (FitSession, model.hpp:118-124).
double objective(sgpx_fit* f, const double* xv, double* gv) {
  ++f->evals;
  ++f->last_step_evals;
  const int64_t ng = f->off_mu;  // beta, variance, l, Z
  f->h_glob.resize(size_t(ng));
  cuok(cudaMemcpyAsync(f->h_glob.data(), xv, sizeof(double) * ng, cudaMemcpyDeviceToHost, f->st), "objective");
  cuok(cudaStreamSynchronize(f->st), "objective");
  const double* hg = f->h_glob.data();
  const double beta = std::exp(hg[0]), var = std::exp(hg[1]);
  std::vector<double> ls(size_t(f->q)), z(size_t(f->m * f->q));
  for (int64_t j = 0; j < f->q; ++j) ls[size_t(j)] = std::exp(hg[2 + j]);
  for (int64_t i = 0; i < f->m; ++i)
    for (int64_t j = 0; j < f->q; ++j) z[size_t(i + j * f->m)] = hg[f->off_z + i * f->q + j];
  sgpx_kernel_spec ks{var, ls.data(), f->q};
  sgpx_cmat zc{z.data(), f->m, f->q, f->m};
  sgpx_cmat muc{}, sc{};
  if (f->latent) {
    exp_kernel<<<grid_for(f->n * f->q), 256, 0, f->st>>>(f->n * f->q, xv + f->off_s, f->sdev);
    g_tc_launches.fetch_add(1);
    cuok(cudaStreamSynchronize(f->st), "objective");  // the engine reads S on its own stream
    muc = sgpx_cmat{xv + f->off_mu, f->n, f->q, f->n};
    sc = sgpx_cmat{f->sdev, f->n, f->q, f->n};
  }
  api(sgpx_engine_broadcast(f->eng, &ks, beta, zc, muc, sc, 1));
  std::vector<double> dz(size_t(f->m * f->q)), dls(size_t(f->q));
  sgpx_eval_result r{};
  r.d_z = dz.data();
  r.d_lengthscales = dls.data();
  const int rc = sgpx_engine_evaluate(f->eng, 1, &r);
  if (rc == SGPX_NUMERIC)
    throw FitError("iteration " + std::to_string(f->iter) + ": " + std::string(sgpx_last_error()));
  api(rc);
  // globals of -pack_gradient (optimizer.hpp:126-144), Z row-major
  std::vector<double> gg(static_cast<size_t>(ng));
  gg[0] = -beta * r.d_beta;
  gg[1] = -var * r.d_variance;
  for (int64_t j = 0; j < f->q; ++j) gg[size_t(2 + j)] = -ls[size_t(j)] * dls[size_t(j)];
  for (int64_t i = 0; i < f->m; ++i)
    for (int64_t j = 0; j < f->q; ++j) gg[size_t(f->off_z + i * f->q + j)] = -dz[size_t(i + j * f->m)];
  cuok(cudaMemcpyAsync(gv, gg.data(), sizeof(double) * ng, cudaMemcpyHostToDevice, f->st), "objective");
  if (f->latent) {
    double *dmu = nullptr, *ds = nullptr;
    api(sgpx_engine_local_grads_device(f->eng, &dmu, &ds));
    local_grad_kernel<<<grid_for(f->n * f->q), 256, 0, f->st>>>(f->n * f->q, dmu, ds, f->sdev, gv + f->off_mu,
                                                               gv + f->off_s);
    g_tc_launches.fetch_add(1);
  }
  cuok(cudaStreamSynchronize(f->st), "objective");  // gg is a stack buffer
  return -r.bound.total;
}

// phi(a) of the line search: x_out = x + a dir, value and gradient there, dphi = g . dir
double phi_at(sgpx_fit* f, double a, double* dphi) {
  xpad(f, f->x, a, f->dir, f->xn);
  const double v = objective(f, f->xn, f->gt);
  *dphi = dot(f, f->gt, f->dir);
  return v;
}

void accept_trial(sgpx_fit* f) { copy(f, f->gn, f->gt); }

// zoom (optimizer.hpp:376-441); on success x_new = xn, g_new = gn
bool zoom(sgpx_fit* f, double f0, double slope0, double alpha_lo, double f_lo, double dphi_lo, double alpha_hi,
          double f_hi, double dphi_hi, double* alpha_out, double* f_out) {
  const double c1 = f->o.c1, c2 = f->o.c2;
  for (int it = 0; it < f->o.max_line_search; ++it) {
    if (f->o.max_evals > 0 && f->evals >= f->o.max_evals) return false;
    double alpha = 0.0;
    {
      const double d1 = dphi_lo + dphi_hi - 3.0 * (f_lo - f_hi) / (alpha_lo - alpha_hi);
      const double disc = d1 * d1 - dphi_lo * dphi_hi;
      if (disc > 0.0) {
        const double d2 = std::sqrt(disc) * (alpha_hi > alpha_lo ? 1.0 : -1.0);
        alpha = alpha_hi - (alpha_hi - alpha_lo) * (dphi_hi + d2 - d1) / (dphi_hi - dphi_lo + 2.0 * d2);
      }
      const double lo = std::min(alpha_lo, alpha_hi), hi = std::max(alpha_lo, alpha_hi);
      const double width = hi - lo;
      if (!(alpha > lo + 0.05 * width && alpha < hi - 0.05 * width)) alpha = 0.5 * (alpha_lo + alpha_hi);
    }
    double dphi = 0.0;
    const double fa = phi_at(f, alpha, &dphi);
    if (!std::isfinite(fa) || fa > f0 + c1 * alpha * slope0 || fa >= f_lo) {
      alpha_hi = alpha;
      f_hi = fa;
      dphi_hi = dphi;
    } else {
      if (std::abs(dphi) <= -c2 * slope0) {
        *alpha_out = alpha;
        *f_out = fa;
        accept_trial(f);
        return true;
      }
      if (dphi * (alpha_hi - alpha_lo) >= 0.0) {
        alpha_hi = alpha_lo;
        f_hi = f_lo;
        dphi_hi = dphi_lo;
      }
      alpha_lo = alpha;
      f_lo = fa;
      dphi_lo = dphi;
    }
    if (std::abs(alpha_hi - alpha_lo) < 1e-16 * std::max(1.0, std::abs(alpha_lo))) break;
  }
  if (f_lo < f0 && alpha_lo > 0.0) {
    double dphi = 0.0;
    *f_out = phi_at(f, alpha_lo, &dphi);
    accept_trial(f);
    *alpha_out = alpha_lo;
    return std::isfinite(*f_out) && *f_out < f0;
  }
  return false;
}

// strong-Wolfe line search (optimizer.hpp:322-373)
bool line_search(sgpx_fit* f, double slope0, double alpha0, double* alpha_out, double* f_out) {
  f->last_step_evals = 0;
  const double f0 = f->value, c1 = f->o.c1, c2 = f->o.c2, alpha_max = 1e10;
  double alpha_prev = 0.0, f_prev = f0, dphi_prev = slope0, alpha = alpha0;
  for (int it = 0; it < f->o.max_line_search; ++it) {
    if (f->o.max_evals > 0 && f->evals >= f->o.max_evals) return false;
    double dphi = 0.0;
    const double fa = phi_at(f, alpha, &dphi);
    if (!std::isfinite(fa)) {
      alpha = 0.5 * (alpha_prev + alpha);
      continue;
    }
    if (fa > f0 + c1 * alpha * slope0 || (it > 0 && fa >= f_prev))
      return zoom(f, f0, slope0, alpha_prev, f_prev, dphi_prev, alpha, fa, dphi, alpha_out, f_out);
    if (std::abs(dphi) <= -c2 * slope0) {
      *alpha_out = alpha;
      *f_out = fa;
      accept_trial(f);
      return true;
    }
    if (dphi >= 0.0) return zoom(f, f0, slope0, alpha, fa, dphi, alpha_prev, f_prev, dphi_prev, alpha_out, f_out);
    alpha_prev = alpha;
    f_prev = fa;
    dphi_prev = dphi;
    alpha = std::min(2.0 * alpha, alpha_max);
    if (alpha >= alpha_max) return false;
  }
  return false;
}

void finish(sgpx_fit* f, int s) {
  f->done = true;
  f->status = s;
}

// LbfgsState::step (optimizer.hpp:243-318)
bool step(sgpx_fit* f) {
  if (f->done) return false;
  const double gn = std::sqrt(dot(f, f->g, f->g));
  if (gn <= f->o.g_tol) {
    finish(f, SGPX_FIT_GRADIENT_CONVERGED);
    return false;
  }
  if (f->o.max_iters >= 0 && f->iter >= f->o.max_iters) {
    finish(f, SGPX_FIT_MAX_ITERATIONS);
    return false;
  }
  if (f->o.max_evals > 0 && f->evals >= f->o.max_evals) {
    finish(f, SGPX_FIT_MAX_EVALUATIONS);
    return false;
  }
  // two-loop recursion
  copy(f, f->dir, f->g);
  axpby(f, 0.0, f->g, -1.0, f->dir);  // dir = -g
  if (!f->hist.empty()) {
    std::vector<double> alpha(f->hist.size());
    for (int64_t i = int64_t(f->hist.size()) - 1; i >= 0; --i) {
      const auto& h = f->hist[size_t(i)];
      alpha[size_t(i)] = h.rho * dot(f, f->hs[size_t(h.slot)], f->dir);
      axpby(f, -alpha[size_t(i)], f->hy[size_t(h.slot)], 1.0, f->dir);
    }
    const auto& last = f->hist.back();
    const double sy = dot(f, f->hs[size_t(last.slot)], f->hy[size_t(last.slot)]);
    const double yy = dot(f, f->hy[size_t(last.slot)], f->hy[size_t(last.slot)]);
    axpby(f, 0.0, f->dir, sy / yy, f->dir);
    for (size_t i = 0; i < f->hist.size(); ++i) {
      const auto& h = f->hist[i];
      const double b = h.rho * dot(f, f->hy[size_t(h.slot)], f->dir);
      axpby(f, alpha[i] - b, f->hs[size_t(h.slot)], 1.0, f->dir);
    }
  }
  double slope = dot(f, f->g, f->dir);
  if (slope >= 0.0) {  // curvature memory went bad: steepest descent
    for (const auto& h : f->hist) f->free_slots.push_back(h.slot);
    f->hist.clear();
    axpby(f, -1.0, f->g, 0.0, f->dir);
    slope = dot(f, f->g, f->dir);
  }
  const double alpha0 = f->hist.empty() ? std::min(1.0, 1.0 / std::max(1.0, gn)) : 1.0;
  double alpha = 0.0, fnew = 0.0;
  if (!line_search(f, slope, alpha0, &alpha, &fnew)) {
    if (f->o.max_evals > 0 && f->evals >= f->o.max_evals) {
      finish(f, SGPX_FIT_MAX_EVALUATIONS);
    } else {
      finish(f, SGPX_FIT_LINE_SEARCH_FAILED);
      f->message = "line search failed to satisfy the Wolfe conditions; returning best iterate";
    }
    return false;
  }
  // s = x_new - x, y = g_new - g into a history slot
  int slot;
  if (!f->free_slots.empty()) {
    slot = f->free_slots.back();
    f->free_slots.pop_back();
  } else if (int(f->hs.size()) < f->o.memory + 1) {
    double *a = nullptr, *b = nullptr;
    cuok(cudaMalloc(&a, sizeof(double) * f->dim), "history");
    cuok(cudaMalloc(&b, sizeof(double) * f->dim), "history");
    f->hs.push_back(a);
    f->hy.push_back(b);
    slot = int(f->hs.size()) - 1;
  } else {
    throw FitError("history slot accounting");
  }
  double* s = f->hs[size_t(slot)];
  double* yv = f->hy[size_t(slot)];
  copy(f, s, f->xn);
  axpby(f, -1.0, f->x, 1.0, s);
  copy(f, yv, f->gn);
  axpby(f, -1.0, f->g, 1.0, yv);
  const double sy = dot(f, s, yv);
  const double sn = std::sqrt(dot(f, s, s)), yn = std::sqrt(dot(f, yv, yv));
  if (sy > 1e-16 * sn * yn) {
    f->hist.push_back({slot, 1.0 / sy});
    if (int(f->hist.size()) > f->o.memory) {
      f->free_slots.push_back(f->hist.front().slot);
      f->hist.pop_front();
    }
  } else {
    f->free_slots.push_back(slot);
  }
  const double f_prev = f->value;
  copy(f, f->x, f->xn);
  copy(f, f->g, f->gn);
  f->value = fnew;
  ++f->iter;
  const double gnew = std::sqrt(dot(f, f->g, f->g));
  if (gnew <= f->o.g_tol) {
    finish(f, SGPX_FIT_GRADIENT_CONVERGED);
  } else if (std::abs(f_prev - f->value) <=
             f->o.f_tol * std::max({std::abs(f_prev), std::abs(f->value), 1.0})) {
    finish(f, SGPX_FIT_VALUE_CONVERGED);
  }
  return true;
}

thread_local std::string g_fit_error;

template <class F>
int fguard(F&& fn) {
  try {
    fn();
    return SGPX_OK;
  } catch (const FitError& e) {
    g_fit_error = e.what();
    const std::string m = e.what();
    return m.rfind("iteration ", 0) == 0 ? SGPX_NUMERIC : SGPX_INTERNAL;
  } catch (const std::exception& e) {
    g_fit_error = e.what();
    return SGPX_INTERNAL;
  }
}

}  // namespace

extern "C" {

void sgpx_lbfgs_default_options(sgpx_lbfgs_options* o) {
  if (!o) return;
  *o = sgpx_lbfgs_options{10, 1e-4, 0.9, 1e-5, 1e-9, 500, 0, 40};
}

const char* sgpx_fit_last_error(void) { return g_fit_error.c_str(); }

int sgpx_fit_create(sgpx_engine* eng, int64_t n_local, const sgpx_kernel_spec* kernel, double beta, sgpx_cmat z,
                    sgpx_cmat mu, sgpx_cmat s, const sgpx_lbfgs_options* opts, sgpx_fit** out) {
  return fguard([&] {
    if (!eng || !kernel || !out) throw FitError("fit_create: null argument");
    if (!(beta > 0.0)) throw FitError("pack: beta must be positive");
    auto f = std::make_unique<sgpx_fit>();
    f->eng = eng;
    f->q = kernel->q;
    f->m = z.rows;
    f->n = n_local;
    f->latent = mu.data != nullptr;
    if (z.cols != f->q) throw FitError("pack: layout mismatch");
    if (opts) f->o = *opts;
    else sgpx_lbfgs_default_options(&f->o);
    f->off_z = 2 + f->q;
    f->off_mu = f->off_z + f->m * f->q;
    f->off_s = f->off_mu + (f->latent ? f->n * f->q : 0);
    f->dim = f->off_s + (f->latent ? f->n * f->q : 0);
    cuok(cudaStreamCreateWithFlags(&f->st, cudaStreamNonBlocking), "stream");
    for (double** p : {&f->x, &f->g, &f->dir, &f->xn, &f->gn, &f->gt})
      cuok(cudaMalloc(p, sizeof(double) * std::max<int64_t>(f->dim, 1)), "fit buffers");
    cuok(cudaMalloc(&f->sdev, sizeof(double) * std::max<int64_t>(f->n * f->q, 1)), "fit buffers");
    cuok(cudaMalloc(&f->part, sizeof(double) * kDotBlocks), "fit buffers");
    cuok(cudaMalloc(&f->scal, sizeof(double)), "fit buffers");
    cuok(cudaMallocHost(&f->h_scal, sizeof(double)), "fit buffers");
    // pack (optimizer.hpp:69-93)
    std::vector<double> glob(static_cast<size_t>(f->off_mu));
    glob[0] = std::log(beta);
    if (!(kernel->variance > 0.0)) throw FitError("kernel variance must be positive");
    glob[1] = std::log(kernel->variance);
    for (int64_t j = 0; j < f->q; ++j) {
      if (!(kernel->lengthscales[j] > 0.0)) throw FitError("kernel lengthscales must be positive");
      glob[size_t(2 + j)] = std::log(kernel->lengthscales[j]);
    }
    const int64_t ldz = z.ld ? z.ld : z.rows;
    for (int64_t i = 0; i < f->m; ++i)
      for (int64_t j = 0; j < f->q; ++j) glob[size_t(f->off_z + i * f->q + j)] = z.data[i + j * ldz];
    cuok(cudaMemcpy(f->x, glob.data(), sizeof(double) * glob.size(), cudaMemcpyHostToDevice), "pack");
    if (f->latent) {
      if (mu.rows != f->n || mu.cols != f->q || s.rows != f->n || s.cols != f->q)
        throw FitError("pack: mu shape mismatch");
      const int64_t ldm = mu.ld ? mu.ld : mu.rows, lds = s.ld ? s.ld : s.rows;
      std::vector<double> ls_host(size_t(f->n * f->q));
      for (int64_t j = 0; j < f->q; ++j)
        for (int64_t i = 0; i < f->n; ++i) {
          const double sv = s.data[i + j * lds];
          if (!(sv > 0.0)) throw FitError("pack: s must be positive");
          ls_host[size_t(i + j * f->n)] = std::log(sv);
        }
      cuok(cudaMemcpy2D(f->x + f->off_mu, sizeof(double) * f->n, mu.data, sizeof(double) * ldm, sizeof(double) * f->n,
                        f->q, cudaMemcpyHostToDevice),
           "pack");
      cuok(cudaMemcpy(f->x + f->off_s, ls_host.data(), sizeof(double) * ls_host.size(), cudaMemcpyHostToDevice),
           "pack");
    }
    // the engine works on the fit's stream
    // (sgpx_ctx_set_stream would change the caller's context; the fit synchronises around calls instead)
    f->value = objective(f.get(), f->x, f->g);  // LbfgsState::initialize (optimizer.hpp:215-221)
    if (!std::isfinite(f->value)) throw FitError("minimize: non-finite objective at start");
    *out = f.release();
  });
}

int sgpx_fit_step(sgpx_fit* f, int* advanced) {
  return fguard([&] {
    if (!f) throw FitError("fit is null");
    f->last_step_evals = 0;
    const bool adv = step(f);
    if (advanced) *advanced = adv ? 1 : 0;
  });
}

int sgpx_fit_state(const sgpx_fit* f, double* value, double* grad_norm, int* iterations, int* total_evals,
                   int* last_step_evals, int* status) {
  return fguard([&] {
    if (!f) throw FitError("fit is null");
    if (value) *value = f->value;
    if (grad_norm) *grad_norm = std::sqrt(dot(const_cast<sgpx_fit*>(f), f->g, f->g));
    if (iterations) *iterations = f->iter;
    if (total_evals) *total_evals = f->evals;
    if (last_step_evals) *last_step_evals = f->last_step_evals;
    if (status) *status = f->done ? f->status : SGPX_FIT_RUNNING;
  });
}

const char* sgpx_fit_message(const sgpx_fit* f) { return f ? f->message.c_str() : ""; }

int sgpx_fit_params(const sgpx_fit* f, double* variance, double* lengthscales, double* beta, sgpx_mmat z,
                    sgpx_mmat mu, sgpx_mmat s) {
  return fguard([&] {
    if (!f) throw FitError("fit is null");
    std::vector<double> glob(static_cast<size_t>(f->off_mu));
    cuok(cudaMemcpy(glob.data(), f->x, sizeof(double) * glob.size(), cudaMemcpyDeviceToHost), "unpack");
    if (beta) *beta = std::exp(glob[0]);
    if (variance) *variance = std::exp(glob[1]);
    if (lengthscales)
      for (int64_t j = 0; j < f->q; ++j) lengthscales[j] = std::exp(glob[size_t(2 + j)]);
    if (z.data) {
      const int64_t ld = z.ld ? z.ld : z.rows;
      for (int64_t i = 0; i < f->m; ++i)
        for (int64_t j = 0; j < f->q; ++j) z.data[i + j * ld] = glob[size_t(f->off_z + i * f->q + j)];
    }
    if (f->latent && mu.data) {
      const int64_t ld = mu.ld ? mu.ld : mu.rows;
      cuok(cudaMemcpy2D(mu.data, sizeof(double) * ld, f->x + f->off_mu, sizeof(double) * f->n, sizeof(double) * f->n,
                        f->q, cudaMemcpyDeviceToHost),
           "unpack");
    }
    if (f->latent && s.data) {
      std::vector<double> tmp(size_t(f->n * f->q));
      cuok(cudaMemcpy(tmp.data(), f->x + f->off_s, sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost), "unpack");
      const int64_t ld = s.ld ? s.ld : s.rows;
      for (int64_t j = 0; j < f->q; ++j)
        for (int64_t i = 0; i < f->n; ++i) s.data[i + j * ld] = std::exp(tmp[size_t(i + j * f->n)]);
    }
  });
}

int sgpx_fit_destroy(sgpx_fit* f) {
  return fguard([&] {
    if (!f) return;
    if (f->st) cudaStreamDestroy(f->st);
    delete f;
  });
}

}  // extern "C"
