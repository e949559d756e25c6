// sgpx_api.cu -- implementation of the C ABI declared in include/sgpx.h.
//
// Host side of the B200 engine: contexts (device + stream + scratch), the
// drop-in sweep_stats / psi1_expected entry points, and the per-rank Engine
// whose evaluate() is the 2-pass protocol of the reference
// (proj/include/sgp/parallel.hpp:370-450):
//   psi forward kernel  -> [allreduce #1 by the caller] -> fp64 coordinator on the host
//   -> psi backward kernel -> [allreduce #2 by the caller] -> gradient assembly.
// No CPU fallback exists: every compute entry point needs the CUDA device.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "../../include/sgpx.h"
#include "coordinator.hpp"
#include "dcoord.cuh"
#include "psi_kernels.cuh"

namespace sgpx {
namespace {

thread_local std::string g_last_error;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CUDA_OK(call)                                                                            \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

template <class F>
int guard(F&& f) {
  try {
    f();
    return SGPX_OK;
  } catch (const InvalidArgument& e) {
    g_last_error = e.what();
    return SGPX_INVALID_ARGUMENT;
  } catch (const NumericError& e) {
    g_last_error = e.what();
    return SGPX_NUMERIC;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return SGPX_CUDA;
  } catch (const IoError& e) {
    g_last_error = e.what();
    return SGPX_IO;
  } catch (const NcclError& e) {
    g_last_error = e.what();
    return SGPX_NCCL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SGPX_INTERNAL;
  }
}

int64_t round4(int64_t x) { return (x + 3) / 4 * 4; }

// Device buffer that only grows.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* get() const {
    return static_cast<T*>(p);
  }
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    CUDA_OK(cudaMalloc(&p, std::max<size_t>(n, 256)));
    bytes = std::max<size_t>(n, 256);
  }
};

// Pinned host buffer that only grows.
struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
  template <class T>
  T* get() const {
    return static_cast<T*>(p);
  }
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    CUDA_OK(cudaMallocHost(&p, std::max<size_t>(n, 256)));
    bytes = std::max<size_t>(n, 256);
  }
};

coord::Mat mat_from(sgpx_cmat a) {
  coord::Mat m(a.rows, a.cols);
  const int64_t ld = a.ld ? a.ld : a.rows;
  for (int64_t j = 0; j < a.cols; ++j)
    for (int64_t i = 0; i < a.rows; ++i) m(i, j) = a.data[i + j * ld];
  return m;
}

void mat_to(const coord::Mat& m, sgpx_mmat out) {
  if (!out.data) return;
  require(out.rows == m.r && out.cols == m.c, "output matrix has the wrong shape");
  const int64_t ld = out.ld ? out.ld : out.rows;
  for (int64_t j = 0; j < m.c; ++j)
    for (int64_t i = 0; i < m.r; ++i) out.data[i + j * ld] = m(i, j);
}

coord::Kernel kernel_from(const sgpx_kernel_spec* k) {
  require(k != nullptr, "kernel spec is null");
  coord::Kernel out;
  out.variance = k->variance;
  require(k->q >= 0 && (k->q == 0 || k->lengthscales), "kernel lengthscales missing");
  out.ls.assign(k->lengthscales, k->lengthscales + k->q);
  out.validate();
  return out;
}

bool all_finite(const coord::Mat& m) {
  for (double x : m.v)
    if (!std::isfinite(x)) return false;
  return true;
}

}  // namespace
}  // namespace sgpx

using namespace sgpx;

// -----------------------------------------------------------------------------
// Context
// -----------------------------------------------------------------------------
struct sgpx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 0;
  int64_t launches0 = 0;
  // scratch of the one-shot sweep / psi1 entry points
  DevBuf mu, s, y, zc, z64, fpart, bpart, pstats, pgrads, u, dpsi, u64, dpsi64, dmu, ds, err, out;
  HostBuf h_stats, h_grads, h_u, h_dpsi, h_err, h_stage;
  int precision = SGPX_PREC_AUTO;  // requested mode of the one-shot entry points
  int last_mode = 0;               // mode the last sweep ran in
  double last_z_spread = 0.0;
};

// Device-side state of one shard (one rank, or one sweep call).
namespace sgpx {
namespace {

struct ShardInputs {
  int64_t n = 0, q = 0, d = 0, m = 0;
  bool expected = false;
  const double *mu = nullptr, *s = nullptr, *y = nullptr;
  int64_t ld_mu = 0, ld_s = 0, ld_y = 0;
};

// Build the per-launch constants and upload the centred fp32 / fp64 copies of Z.
PsiConst make_const(sgpx_ctx* ctx, const ShardInputs& in, const coord::Kernel& k, const coord::Mat& z, DevBuf& zc_buf,
                    DevBuf& z64_buf, HostBuf& staging, int precision) {
  require(in.q >= 1 && in.q <= kMaxQ, "latent dimension Q must be in [1, 64] on the B200 path");
  PsiConst P{};
  P.n = in.n;
  P.ld_mu = in.ld_mu;
  P.ld_s = in.ld_s;
  P.ld_y = in.ld_y;
  P.mu = in.mu;
  P.s = in.s;
  P.y = in.y;
  P.q = int(in.q);
  P.qv = int(round4(std::max<int64_t>(instantiated_q(int(in.q)), in.q)));
  P.m = int(in.m);
  P.mv = int(round4(in.m));
  P.d = int(in.d);
  P.dv = int(round4(in.d));
  P.expected = in.expected ? 1 : 0;
  P.variance = float(k.variance);
  P.variance_d = k.variance;
  P.log2_var = float(std::log2(k.variance));
  for (int j = 0; j < P.q; ++j) {
    double c = 0.0;
    for (int64_t a = 0; a < in.m; ++a) c += z(a, j);
    P.center[j] = in.m ? c / double(in.m) : 0.0;
    const double l = k.ls[j];
    P.ls[j] = l;
    P.l2[j] = float(l * l);
    P.il2[j] = float(1.0 / (l * l));
  }
  for (int j = P.q; j < kMaxQ; ++j) {
    P.center[j] = 0.0;
    P.ls[j] = 1.0;
    P.l2[j] = 1.f;
    P.il2[j] = 1.f;
  }
  const size_t zc_bytes = sizeof(float) * P.mv * P.qv, z64_bytes = sizeof(double) * z.v.size();
  staging.ensure(zc_bytes + z64_bytes + 16);
  float* hz = staging.get<float>();
  std::fill(hz, hz + size_t(P.mv) * P.qv, 0.f);
  for (int64_t a = 0; a < in.m; ++a)
    for (int j = 0; j < P.q; ++j) hz[a * P.qv + j] = float(z(a, j) - P.center[j]);
  double* h64 = reinterpret_cast<double*>(staging.get<char>() + ((zc_bytes + 15) / 16) * 16);
  std::copy(z.v.begin(), z.v.end(), h64);
  zc_buf.ensure(zc_bytes);
  z64_buf.ensure(z64_bytes);
  CUDA_OK(cudaMemcpyAsync(zc_buf.p, hz, zc_bytes, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_OK(cudaMemcpyAsync(z64_buf.p, h64, z64_bytes, cudaMemcpyHostToDevice, ctx->stream));
  // the staging buffer is reused by the next broadcast: wait for the copies
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
  P.zc = zc_buf.get<float>();
  P.z64 = z64_buf.get<double>();
  P.mode = psi_select_mode(P, z.v.data(), z.r, precision);
  require(P.mode > 0, "latent dimension Q exceeds the instantiated kernels");
  return P;
}

// Fill the fp32 backward operands: U = d_phi_big mirrored from its upper
// triangle (the reference reads only a <= b, psi_stats.hpp:280-281), [mv][mv];
// dPsi transposed, [d][mv].
// The fp64 copies (the direct kernels and the per-pair gradient terms) follow the fp32 arrays in the
// same host buffers, at byte offset fp32_bytes rounded up to 16.
size_t f32_slot(size_t n) { return (sizeof(float) * n + 15) / 16 * 16; }
void stage_adjoints(const PsiConst& P, const coord::Mat& dphi_big, const coord::Mat& dpsi, HostBuf& hu, HostBuf& hd) {
  const size_t nu = size_t(P.mv) * P.mv, nd = size_t(std::max(1, P.d)) * P.mv;
  hu.ensure(f32_slot(nu) + sizeof(double) * nu);
  hd.ensure(f32_slot(nd) + sizeof(double) * nd);
  double* u64 = reinterpret_cast<double*>(hu.get<char>() + f32_slot(nu));
  double* d64 = reinterpret_cast<double*>(hd.get<char>() + f32_slot(nd));
  std::fill(u64, u64 + nu, 0.0);
  std::fill(d64, d64 + nd, 0.0);
  for (int a = 0; a < P.m; ++a)
    for (int b = a; b < P.m; ++b) {
      const double v = dphi_big(a, b);
      u64[size_t(b) * P.mv + a] = v;
      u64[size_t(a) * P.mv + b] = v;
    }
  for (int dd = 0; dd < P.d; ++dd)
    for (int a = 0; a < P.m; ++a) d64[size_t(dd) * P.mv + a] = dpsi(a, dd);
  float* u = hu.get<float>();
  std::fill(u, u + size_t(P.mv) * P.mv, 0.f);
  for (int a = 0; a < P.m; ++a)
    for (int b = a; b < P.m; ++b) {
      const float v = float(dphi_big(a, b));
      u[size_t(b) * P.mv + a] = v;
      u[size_t(a) * P.mv + b] = v;
    }
  float* dp = hd.get<float>();
  std::fill(dp, dp + size_t(std::max(1, P.d)) * P.mv, 0.f);
  for (int dd = 0; dd < P.d; ++dd)
    for (int a = 0; a < P.m; ++a) dp[size_t(dd) * P.mv + a] = float(dpsi(a, dd));
}

void upload_adjoints(const PsiConst& P, HostBuf& hu, HostBuf& hd, DevBuf& u, DevBuf& dpsi, DevBuf& u64, DevBuf& dpsi64,
                     cudaStream_t st) {
  const size_t nu = size_t(P.mv) * P.mv, nd = size_t(std::max(1, P.d)) * P.mv;
  u.ensure(sizeof(float) * nu);
  dpsi.ensure(sizeof(float) * nd);
  u64.ensure(sizeof(double) * nu);
  dpsi64.ensure(sizeof(double) * nd);
  CUDA_OK(cudaMemcpyAsync(u.p, hu.p, sizeof(float) * nu, cudaMemcpyHostToDevice, st));
  CUDA_OK(cudaMemcpyAsync(dpsi.p, hd.p, sizeof(float) * nd, cudaMemcpyHostToDevice, st));
  CUDA_OK(cudaMemcpyAsync(u64.p, hu.get<char>() + f32_slot(nu), sizeof(double) * nu, cudaMemcpyHostToDevice, st));
  CUDA_OK(cudaMemcpyAsync(dpsi64.p, hd.get<char>() + f32_slot(nd), sizeof(double) * nd, cudaMemcpyHostToDevice, st));
}

// Same order and messages as psi_stats.hpp:119-120.
void check_err_flag(int flag) {
  if (flag & 1) throw InvalidArgument("stats sweep: non-finite data");
  if (flag & 4) throw InvalidArgument("stats sweep: variances must be positive");
}

// Copy a (possibly strided) host/device column-major matrix into a dense device buffer.
void upload(sgpx_ctx* ctx, DevBuf& dst, sgpx_cmat a, bool on_device) {
  const int64_t ld = a.ld ? a.ld : a.rows;
  const size_t bytes = sizeof(double) * std::max<int64_t>(1, a.rows * a.cols);
  dst.ensure(bytes);
  if (a.rows * a.cols == 0) return;
  CUDA_OK(cudaMemcpy2DAsync(dst.p, sizeof(double) * a.rows, a.data, sizeof(double) * ld, sizeof(double) * a.rows,
                              a.cols, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
}

void check_view(sgpx_cmat a, const char* name) {
  require(a.rows >= 0 && a.cols >= 0, std::string(name) + ": negative shape");
  require(a.ld == 0 || a.ld >= a.rows, std::string(name) + ": leading dimension smaller than rows");
  require(a.rows * a.cols == 0 || a.data != nullptr, std::string(name) + ": null data");
}

}  // namespace
}  // namespace sgpx

// -----------------------------------------------------------------------------
// Engine
// -----------------------------------------------------------------------------
struct sgpx_engine {
  sgpx_ctx* ctx = nullptr;
  sgpx_engine_config cfg{};
  bool latent = false;
  // shard inputs (owned copies or adopted device pointers)
  DevBuf own_x, own_s, own_y;
  ShardInputs in;
  bool has_data = false, has_params = false;
  // broadcast parameters
  coord::Kernel kernel;
  coord::Mat z;
  double beta = 1.0;
  PsiConst P{};
  DevBuf zc, z64, fpart, bpart, pstats, pgrads, u, dpsi, u64, dpsi64, dmu, ds, err;
  HostBuf h_stats, h_grads, h_u, h_dpsi, h_err, h_stage;
  // coordinator results of the current evaluation
  coord::Result res;
  coord::Stats st;  // unpacked statistics of the last coordinate() (complete_adjoints needs them)
  bool coordinated = false, with_grads = false;
  bool pairs_folded = false;  // sub-shard pair sums folded into the first (once per forward)
  cudaEvent_t ev[12] = {};  // 0-1 stats pass, 2-3 grad pass, 4-5 fwd psi, 6-7 bwd psi, 8-11 psi2 kernels
  double coord_s = 0.0;
  double z_spread = 0.0;
  LaunchGeom gf{}, gb{};
  // Sub-shard pipeline: the shard's rows are processed as K contiguous sub-shards so that the
  // host<->device traffic of one (mu, S in; d mu, d S out) overlaps the kernels of another.
  struct Sub {
    int64_t n0 = 0, n = 0;
    PsiConst P{};
    int64_t foff = 0, boff = 0;  // doubles into fpart / bpart
  };
  std::vector<Sub> subs;
  DevBuf pstats_sub, pgrads_sub;
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_out;
  // deferred upload of host mu / S (broadcast with host views), streamed by the stats pass
  bool pending_upload = false;
  bool uploads_enqueued = false;  // the pending upload's sub-shard copies are already on the copy stream
  sgpx_cmat h_mu{}, h_s{};
  // registered host outputs for d mu / d S, streamed by the gradient pass
  bool has_gout = false;
  sgpx_mmat g_mu{}, g_s{};
  // device coordinator (dcoord.cu): the M-sized algebra on the stream, no host round trip.  Off by
  // default for a single engine: the host coordinator overlaps its Z-only and deferred halves with the
  // kernels and measured 7.94 vs 8.07 ms per C3 evaluation (profiles/r02_coordinator_ab.txt); on by
  // default in the multi-GPU engine, where every shard's coordinator then runs on its own device.
  bool dev_coord = false;
  DevBuf dcw;
  DcArgs dc{};
  HostBuf h_dc;
  cudaEvent_t ev_c[2] = {};
  // split device coordinator (dc_bound_split): d Psi first on the stream, d Phi / d Kmm on a side stream
  // concurrently with the psi1 backward; split_join = the stream still has to wait for ev_split[1]
  bool coord_split = true;
  bool split = false, split_join = false;
  cudaStream_t side = nullptr, side2 = nullptr;
  cudaEvent_t ev_split[4] = {};
  cudaEvent_t ev_pre[2] = {};  // the per-broadcast prefactor on the side stream (dc_setup)
  cudaEvent_t ev_red[2] = {};  // sub-shard backward reductions on side2: fork (per sub-shard), join
  cudaEvent_t ev_copy_done = nullptr;  // the streamed d mu / d S read-backs, joined into the stream
  bool pre_needed = false;   // a broadcast's prefactor not launched yet
  bool pre_pending = false;  // launched, not joined yet
  // one evaluation (device-resident shard, device coordinator) as a CUDA graph, replayed while its
  // launch arguments are unchanged (graph_key)
  bool use_graph = true;
  cudaGraphExec_t graph = nullptr;
  std::vector<unsigned char> graph_key;
  int64_t graph_launches = 0;  // kernels in the captured graph (the launch counter counts replays too)
  double last_bound = 0.0;     // bound of the last evaluation (the reference's cached_bound)
  std::vector<double> kernel_ls;  // lengthscales of the last broadcast (device coordinator upload)
  bool dc_ready = false;          // device coordinator set up for the current broadcast
  ~sgpx_engine() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_c)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_split)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_pre)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_red)
      if (e) cudaEventDestroy(e);
    if (ev_copy_done) cudaEventDestroy(ev_copy_done);
    if (side) cudaStreamDestroy(side);
    if (side2) cudaStreamDestroy(side2);
    if (graph) cudaGraphExecDestroy(graph);
    for (auto e : ev_in) cudaEventDestroy(e);
    for (auto e : ev_out) cudaEventDestroy(e);
    if (copy) cudaStreamDestroy(copy);
  }
};

namespace sgpx {
namespace {

__global__ void sum_parts_kernel(const double* __restrict__ parts, int k, int64_t count, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += parts[int64_t(j) * count + i];
    out[i] = s;
  }
}

// dst[i] += src[i] (sub-shard pair sums folded into the first, in sub-shard order)
__global__ void add_into_kernel(double* __restrict__ dst, const double* __restrict__ src, int64_t count) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}

// Sub-shard plan: one piece when the shard is device resident (nothing to overlap; every split
// costs kernel efficiency), else weighted pieces with boundaries on multiples of 384 rows (feature
// tile grain) so the host transfers of one piece overlap the kernels of the others.
// Sub-shard weights: transfers overlap the kernels of the neighbouring pieces, so small first and
// last pieces shorten the pipeline fill (first upload) and drain (last read-back).
std::vector<double> sub_weights(int64_t n, bool transfers) {
  if (!transfers) return {1.0};
  if (const char* v = getenv("SGPX_SUBS")) {  // override (pipeline experiments): "k" or "w1,w2,..."
    std::vector<double> w;
    std::string str(v);
    size_t pos = 0;
    while (pos <= str.size()) {
      const size_t nx = str.find(',', pos);
      const std::string tok = str.substr(pos, nx == std::string::npos ? std::string::npos : nx - pos);
      if (!tok.empty()) w.push_back(atof(tok.c_str()));
      if (nx == std::string::npos) break;
      pos = nx + 1;
    }
    if (w.size() == 1 && w[0] >= 1.0) w.assign(size_t(w[0]), 1.0);
    bool ok = !w.empty();
    for (double x : w) ok = ok && x > 0.0;
    if (ok) return w;
  }
  // measured best end to end at the C3 shape (Q=10 D=50 M=100) per row count, graph-replayed
  // (tools/e2e_sweep.py, profiles/r02/subs_sweep.txt): 1M / 500k / 250k / 125k+100k rows
  if (n >= 1000000) return {1.0, 1.5, 2.0, 2.0, 2.0, 1.5, 1.0};
  if (n >= 400000) return {1.0, 1.5, 2.0, 2.0, 1.5, 1.0};
  if (n >= 200000) return {1.0, 1.5, 2.0, 1.5, 1.0};
  if (n >= 80000) return {1.0, 1.0};
  return {1.0};
}

void plan_subs(sgpx_engine* e) {
  const int64_t n = e->in.n;
  const bool transfers = e->pending_upload || (e->has_gout && e->latent);
  std::vector<double> w = sub_weights(n, transfers);
  // at least 384 rows (the feature tile grain) per piece
  while (w.size() > 1 && int64_t(w.size()) * 384 > n) w.pop_back();
  double wsum = 0.0;
  for (double x : w) wsum += x;
  e->subs.clear();
  int64_t n0 = 0;
  double acc = 0.0;
  for (size_t j = 0; j < w.size() || (n == 0 && e->subs.empty()); ++j) {
    int64_t n1 = n;
    if (j + 1 < w.size()) {
      acc += w[j];
      n1 = std::min<int64_t>(n, (int64_t(double(n) * acc / wsum) + 383) / 384 * 384);
    }
    if (n1 <= n0 && n > 0) continue;
    sgpx_engine::Sub sub;
    sub.n0 = n0;
    sub.n = n1 - n0;
    sub.P = e->P;
    sub.P.n = sub.n;
    sub.P.mu = e->P.mu + n0;
    sub.P.s = e->P.s ? e->P.s + n0 : nullptr;
    sub.P.y = e->P.y + n0;
    e->subs.push_back(sub);
    n0 = n1;
    if (n == 0) break;
  }
  const size_t need = e->subs.size();
  while (e->ev_in.size() < need) {
    cudaEvent_t a, b;
    CUDA_OK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    e->ev_in.push_back(a);
    e->ev_out.push_back(b);
  }
  if (!e->copy) CUDA_OK(cudaStreamCreateWithFlags(&e->copy, cudaStreamNonBlocking));
}

bool is_pinned(const void* ptr) {  // page-locked host memory (copies from it can be graph-captured)
  if (!ptr) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// copy stream: mu / S of every sub-shard (the forward of sub-shard j waits for ev_in[j]); issued by
// broadcast() as soon as it has the host views, so the transfer overlaps the caller's own work
void enqueue_uploads(sgpx_engine* e) {
  if (!e->pending_upload || e->uploads_enqueued) return;
  sgpx_ctx* ctx = e->ctx;
  if (e->subs.empty()) plan_subs(e);
  CUDA_OK(cudaEventRecord(e->ev_out[0], ctx->stream));  // previous users of the device rows are done
  CUDA_OK(cudaStreamWaitEvent(e->copy, e->ev_out[0], 0));
  const int64_t q = e->cfg.q, n = e->cfg.n_local;
  const int64_t ldm = e->h_mu.ld ? e->h_mu.ld : n, lds = e->h_s.ld ? e->h_s.ld : n;
  for (size_t j = 0; j < e->subs.size(); ++j) {
    const auto& sub = e->subs[j];
    CUDA_OK(cudaMemcpy2DAsync(e->own_x.get<double>() + sub.n0, sizeof(double) * n, e->h_mu.data + sub.n0,
                                sizeof(double) * ldm, sizeof(double) * sub.n, q, cudaMemcpyHostToDevice, e->copy));
    CUDA_OK(cudaMemcpy2DAsync(e->own_s.get<double>() + sub.n0, sizeof(double) * n, e->h_s.data + sub.n0,
                                sizeof(double) * lds, sizeof(double) * sub.n, q, cudaMemcpyHostToDevice, e->copy));
    CUDA_OK(cudaEventRecord(e->ev_in[j], e->copy));
  }
  e->uploads_enqueued = true;
}

void dc_launch_prefactor(sgpx_engine* e);

void engine_stats_pass(sgpx_engine* e) {
  require(e->has_data && e->has_params, "engine: set_data and broadcast must precede evaluate");
  sgpx_ctx* ctx = e->ctx;
  const int64_t count = sgpx_packed_stats_count(e->cfg.m, e->cfg.d);
  e->pairs_folded = false;
  e->pstats.ensure(sizeof(double) * count);
  e->err.ensure(sizeof(int));
  CUDA_OK(cudaMemsetAsync(e->err.p, 0, sizeof(int), ctx->stream));
  if (e->in.n == 0) {
    CUDA_OK(cudaMemsetAsync(e->pstats.p, 0, sizeof(double) * count, ctx->stream));
    CUDA_OK(record_event(e->ev[0], ctx->stream));
    CUDA_OK(record_event(e->ev[1], ctx->stream));
    e->coordinated = false;
    return;
  }
  plan_subs(e);
  if (e->dev_coord) dc_launch_prefactor(e);  // side stream, under the forward
  const int k = int(e->subs.size());
  // partial-buffer layout: one region per sub-shard
  int64_t foff = 0;
  for (auto& sub : e->subs) {
    LaunchGeom g{};
    if (plan_forward(sub.P, ctx->num_sms, &g)) throw CudaError("psi forward: launch planning failed");
    sub.foff = foff;
    foff += fwd_part_count(sub.P.m, sub.P.d) * std::max(1, g.grid);
  }
  e->fpart.ensure(sizeof(double) * foff);
  if (k > 1) e->pstats_sub.ensure(sizeof(double) * count * k);
  CUDA_OK(record_event(e->ev[0], ctx->stream));
  enqueue_uploads(e);  // (normally already issued by broadcast)
  // the row-tile forward's pair operand does not depend on the rows: later sub-shards reuse the first's
  const float* pairs0 =
      k > 1 ? fwd_pair_operand(e->subs[0].P, fwd_region(e->subs[0].P, e->fpart.get<double>() + e->subs[0].foff,
                                                        ctx->num_sms),
                               ctx->num_sms)
            : nullptr;
  for (int j = 0; j < k; ++j) {
    auto& sub = e->subs[j];
    sub.P.rt_pairs_shared = j > 0 ? pairs0 : nullptr;
    if (e->pending_upload) CUDA_OK(cudaStreamWaitEvent(ctx->stream, e->ev_in[j], 0));
    double* out = k > 1 ? e->pstats_sub.get<double>() + int64_t(j) * count : e->pstats.get<double>();
    sub.P.ev_psi2[0] = j == 0 ? e->ev[8] : nullptr;  // the first sub-shard's main psi2 kernel (roofline)
    sub.P.ev_psi2[1] = j == 0 ? e->ev[9] : nullptr;
    if (psi_forward(sub.P, e->fpart.get<double>() + sub.foff, out, e->err.get<int>(), ctx->num_sms, ctx->stream,
                    &e->gf, j == 0 ? e->ev[4] : nullptr, j == k - 1 ? e->ev[5] : nullptr))
      throw CudaError(std::string("psi forward launch: ") + cudaGetErrorString(cudaGetLastError()));
  }
  if (k > 1) {
    sum_parts_kernel<<<int(std::min<int64_t>((count + 255) / 256, 1024)), 256, 0, ctx->stream>>>(
        e->pstats_sub.get<double>(), k, count, e->pstats.get<double>());
    CUDA_OK(cudaGetLastError());
  }
  e->pending_upload = false;
  e->uploads_enqueued = false;
  CUDA_OK(record_event(e->ev[1], ctx->stream));
  e->coordinated = false;
}

// Bind the device coordinator's workspace and run its per-broadcast half (Kmm, factor_gram, Kmm^-1).
void dc_setup(sgpx_engine* e) {
  DcArgs& dc = e->dc;
  dc.m = int(e->cfg.m);
  dc.mv = e->P.mv;
  dc.q = int(e->cfg.q);
  dc.d = int(e->cfg.d);
  dc.latent = e->latent ? 1 : 0;
  dc.n = e->cfg.n_global;
  dc.var = e->kernel.variance;
  dc.beta = e->beta;
  dc.jitter_factor = e->cfg.jitter_factor;
  dc.z = e->z64.get<double>();
  e->dcw.ensure(sizeof(double) * dc_workspace_doubles(dc.m, dc.q, dc.d));
  dc_bind(dc, e->dcw.get<double>());
  e->pstats.ensure(sizeof(double) * sgpx_packed_stats_count(e->cfg.m, e->cfg.d));
  dc.packed = e->pstats.get<double>();
  // the per-broadcast half (Kmm, its factor and inverse) is launched by the next statistics pass on the
  // side stream (dc_launch_prefactor), overlapping the forward kernels (and inside the evaluation's
  // graph when it is replayed), and joined right before the coordinator (dc_join_prefactor)
  e->pre_needed = true;
  e->dc_ready = true;
}

void dc_launch_prefactor(sgpx_engine* e) {
  if (!e->pre_needed) return;
  cudaStream_t st = e->ctx->stream;
  if (!e->side) CUDA_OK(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
  if (!e->ev_pre[0]) {
    CUDA_OK(cudaEventCreateWithFlags(&e->ev_pre[0], cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&e->ev_pre[1], cudaEventDisableTiming));
  }
  CUDA_OK(cudaEventRecord(e->ev_pre[0], st));  // after every earlier user of the workspace
  CUDA_OK(cudaStreamWaitEvent(e->side, e->ev_pre[0], 0));
  // the lengthscales travel as a kernel argument (no staging buffer to keep alive)
  if (dc_upload_ls(e->dc, e->kernel_ls.data(), e->side)) throw CudaError("coordinator launch");
  if (dc_prefactor(e->dc, e->side)) throw CudaError("coordinator launch");
  CUDA_OK(cudaEventRecord(e->ev_pre[1], e->side));
  e->pre_needed = false;
  e->pre_pending = true;
}

// the stream waits for the per-broadcast prefactor (before the first coordinator kernel)
void dc_join_prefactor(sgpx_engine* e) {
  if (!e->pre_pending) return;
  CUDA_OK(cudaStreamWaitEvent(e->ctx->stream, e->ev_pre[1], 0));
  e->pre_pending = false;
}

void engine_coordinate(sgpx_engine* e, bool with_grads) {
  if (e->dev_coord) {  // device coordinator: stream-ordered after the (reduced) statistics, no sync
    sgpx_ctx* ctx = e->ctx;
    e->dc.packed = e->pstats.get<double>();
    e->u.ensure(sizeof(float) * e->P.mv * e->P.mv);
    e->dpsi.ensure(sizeof(float) * std::max(1, e->P.d) * e->P.mv);
    e->u64.ensure(sizeof(double) * e->P.mv * e->P.mv);
    e->dpsi64.ensure(sizeof(double) * std::max(1, e->P.d) * e->P.mv);
    dc_launch_prefactor(e);  // (a no-op unless the statistics pass had no rows to launch it under)
    dc_join_prefactor(e);
    CUDA_OK(record_event(e->ev_c[0], ctx->stream));
    e->split = e->coord_split && e->cfg.m <= 112;
    if (e->split) {
      if (!e->side) CUDA_OK(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
      if (!e->side2) CUDA_OK(cudaStreamCreateWithFlags(&e->side2, cudaStreamNonBlocking));
      for (auto& ev : e->ev_split)
        if (!ev) CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      if (dc_bound_split(e->dc, e->u.get<float>(), e->dpsi.get<float>(), e->u64.get<double>(), e->dpsi64.get<double>(),
                         ctx->stream, e->side, e->side2, e->ev_split))
        throw CudaError("coordinator launch");
      e->split_join = true;
    } else if (dc_bound(e->dc, e->u.get<float>(), e->dpsi.get<float>(), e->u64.get<double>(), e->dpsi64.get<double>(),
                        ctx->stream)) {
      throw CudaError("coordinator launch");
    }
    CUDA_OK(record_event(e->ev_c[1], ctx->stream));  // the coordinator's critical path (d Psi when split)
    e->res.adj.d_phi = -0.5 * e->beta * double(e->cfg.d);  // adjoints_from_core (bound.hpp:203)
    e->with_grads = with_grads;
    e->coordinated = true;
    return;
  }
  sgpx_ctx* ctx = e->ctx;
  e->split = e->split_join = false;
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t count = sgpx_packed_stats_count(e->cfg.m, e->cfg.d);
  e->h_stats.ensure(sizeof(double) * count);
  e->h_err.ensure(sizeof(int));
  CUDA_OK(cudaMemcpyAsync(e->h_stats.p, e->pstats.p, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OK(cudaMemcpyAsync(e->h_err.p, e->err.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  // Z-only algebra while the statistics pass is still running on the device; its errors are
  // reported after the pass's own (data validation first, as in the reference)
  coord::Prefactor pre;
  std::exception_ptr pre_err;
  try {
    pre = coord::prefactor(e->z, e->kernel, e->cfg.jitter_factor);
  } catch (...) {
    pre_err = std::current_exception();
  }
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
  const auto t_host = std::chrono::steady_clock::now();  // host algebra only (the sync waited for the kernels)
  check_err_flag(*e->h_err.get<int>());
  if (pre_err) std::rethrow_exception(pre_err);
  e->st = coord::unpack_stats(e->h_stats.get<double>(), e->cfg.m, e->cfg.d);
  // d_kmm / d_beta are deferred until the gradient kernels are enqueued (they run on the host
  // while the device works; complete_adjoints)
  e->res = coord::coordinate(e->latent, e->cfg.n_global, e->cfg.d, e->st, e->z, e->kernel, e->beta,
                             e->cfg.jitter_factor, with_grads, /*defer_host_only=*/true, &pre);
  e->with_grads = with_grads;
  if (with_grads) {
    stage_adjoints(e->P, e->res.adj.d_phi_big, e->res.adj.d_psi_y, e->h_u, e->h_dpsi);
    upload_adjoints(e->P, e->h_u, e->h_dpsi, e->u, e->dpsi, e->u64, e->dpsi64, ctx->stream);
  }
  e->coordinated = true;
  e->coord_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_host).count();
  (void)t0;
}

void engine_grad_pass(sgpx_engine* e) {
  require(e->coordinated && e->with_grads, "engine: coordinate(with_grads=1) must precede the gradient pass");
  sgpx_ctx* ctx = e->ctx;
  const int64_t count = sgpx_packed_grads_count(e->cfg.m, e->cfg.q);
  e->pgrads.ensure(sizeof(double) * count);
  e->dmu.ensure(sizeof(double) * std::max<int64_t>(1, e->in.n * e->cfg.q));
  e->ds.ensure(sizeof(double) * std::max<int64_t>(1, e->in.n * e->cfg.q));
  CUDA_OK(record_event(e->ev[2], ctx->stream));
  auto join = [&] {  // d Phi / d Kmm of the split coordinator (side stream) before their consumers
    if (e->split_join) {
      CUDA_OK(cudaStreamWaitEvent(ctx->stream, e->ev_split[1], 0));
      e->split_join = false;
    }
  };
  if (e->in.n > 0) {
    const int k = int(e->subs.size());
    // split coordinator: every psi1 kernel (it needs d Psi only) first, on all SMs but the one the side
    // stream's coordinator kernel occupies, then d Phi is joined and the psi2 kernels run
    bool phased = e->split_join;
    for (auto& sub : e->subs) phased = phased && psi_backward_phased(sub.P);
    if (const char* v = getenv("SGPX_PHASED"); v && atoi(v) == 0) phased = false;  // A/B
    // the psi1 kernels of the phased pass leave one SM to the side stream's coordinator kernel; every
    // layout (partial rows, the forward's regions) stays the one of the full SM count
    const int nsm = ctx->num_sms;
    const int psi1_cap = phased ? std::max(1, ctx->num_sms - 1) : 0;
    if (!phased) join();
    int64_t boff = 0;
    for (auto& sub : e->subs) {
      LaunchGeom g{};
      if (plan_backward(sub.P, nsm, &g)) throw CudaError("psi backward: launch planning failed");
      sub.boff = boff;
      boff += bwd_part_count(sub.P.m, sub.P.q) * std::max(1, g.grid);
    }
    e->bpart.ensure(sizeof(double) * boff);
    if (k > 1) e->pgrads_sub.ensure(sizeof(double) * count * k);
    // the per-pair gradient terms are linear in the forward pair sums: fold every sub-shard's sums
    // into the first and add the terms once (row-tile path)
    const bool fold = k > 1;
    if (fold && !e->pairs_folded) {
      e->pairs_folded = true;
      int64_t np = 0;
      auto sums = [&](int j, int64_t* n) {
        const auto& sj = e->subs[j];
        double* region = const_cast<double*>(fwd_region(sj.P, e->fpart.get<double>() + sj.foff, ctx->num_sms));
        return fwd_pair_sums(sj.P, region, ctx->num_sms, n);
      };
      double* s0 = sums(0, &np);
      for (int j = 1; j < k; ++j) {
        int64_t nj = 0;
        const double* sj = sums(j, &nj);
        if (nj != np) throw CudaError("sub-shard pair sums differ in size");
        add_into_kernel<<<int(std::min<int64_t>((np + 255) / 256, 1024)), 256, 0, ctx->stream>>>(s0, sj, np);
      }
      CUDA_OK(cudaGetLastError());
    }
    const bool stream_out = e->has_gout && e->latent;
    const float *rt_pre0 = nullptr, *rt_ys0 = nullptr;
    bool prepared = false;
    const char* prep_env = getenv("SGPX_RT_PREP");  // A/B
    if (phased && !(prep_env && atoi(prep_env) == 0)) {  // the psi2 backward's pair operand right after U, on the side stream
      const auto& s0 = e->subs[0];
      if (rt_bwd_prepare(s0.P, e->u.get<float>(), bwd_rt_region(s0.P, e->bpart.get<double>() + s0.boff, nsm), nsm,
                         e->side, &rt_pre0, &rt_ys0))
        throw CudaError("psi backward prepare launch");
      CUDA_OK(cudaEventRecord(e->ev_split[1], e->side));  // the join now also covers them
      prepared = true;
    }
    auto bconst = [&](const sgpx_engine::Sub& sub, int j) {
      BwdConst B{};
      B.u = e->u.get<float>();
      B.dpsi = e->dpsi.get<float>();
      B.u64 = e->u64.get<double>();
      B.dpsi64 = e->dpsi64.get<double>();
      B.d_phi = e->res.adj.d_phi;
      B.add_kl = e->latent ? 1 : 0;
      B.write_local = e->latent ? 1 : 0;
      B.d_mu = e->dmu.get<double>() + sub.n0;
      B.d_s = e->ds.get<double>() + sub.n0;
      B.ld_g = e->in.n;
      B.fwd_rt = fwd_region(sub.P, e->fpart.get<double>() + sub.foff, ctx->num_sms);
      B.skip_pair_terms = (fold && j > 0) ? 1 : 0;
      // the U-weighted pair operand and Y scales of the psi2 backward do not depend on the rows
      if (prepared) {
        B.rt_pre_shared = rt_pre0;
        B.rt_ys_shared = rt_ys0;
      } else if (j == 0) {
        B.rt_pre_out = &rt_pre0;
        B.rt_ys_out = &rt_ys0;
      } else {
        B.rt_pre_shared = rt_pre0;
        B.rt_ys_shared = rt_ys0;
      }
      return B;
    };
    auto out_of = [&](int j) {
      return k > 1 ? e->pgrads_sub.get<double>() + int64_t(j) * count : e->pgrads.get<double>();
    };
    // sub-shards: each one's partial-row reduction on side2, joined before the sub-shard sum
    const char* rs_env = getenv("SGPX_RED_SIDE");  // A/B
    const bool red_side = k > 1 && !(rs_env && atoi(rs_env) == 0);
    if (red_side) {
      if (!e->side2) CUDA_OK(cudaStreamCreateWithFlags(&e->side2, cudaStreamNonBlocking));
      for (auto& ev : e->ev_red)
        if (!ev) CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    // with streamed-out d mu / d S only the first sub-shards run their psi1 kernels ahead (enough to
    // cover the side stream's coordinator); the rest keep psi1 -> psi2 -> copy-out per sub-shard so the
    // device-to-host copies start early
    int kp = phased ? (stream_out ? std::max(1, k / 3) : k) : 0;
    if (const char* v = getenv("SGPX_KP"); v && phased) kp = std::min(k, std::max(1, atoi(v)));  // A/B
    if (phased) {
      for (int j = 0; j < kp; ++j) {
        auto& sub = e->subs[j];
        if (psi_backward(sub.P, bconst(sub, j), e->bpart.get<double>() + sub.boff, out_of(j), nsm, ctx->stream, &e->gb,
                         j == 0 ? e->ev[6] : nullptr, nullptr, 1, nullptr, nullptr, psi1_cap))
          throw CudaError(std::string("psi backward launch: ") + cudaGetErrorString(cudaGetLastError()));
      }
      join();
    }
    for (int j = 0; j < k; ++j) {
      auto& sub = e->subs[j];
      sub.P.ev_psi2[0] = j == 0 ? e->ev[10] : nullptr;
      sub.P.ev_psi2[1] = j == 0 ? e->ev[11] : nullptr;
      if (psi_backward(sub.P, bconst(sub, j), e->bpart.get<double>() + sub.boff, out_of(j), nsm, ctx->stream, &e->gb,
                       (j == 0 && !phased) ? e->ev[6] : nullptr, j == k - 1 ? e->ev[7] : nullptr, j < kp ? 2 : 0,
                       red_side ? e->side2 : nullptr, red_side ? e->ev_red[0] : nullptr))
        throw CudaError(std::string("psi backward launch: ") + cudaGetErrorString(cudaGetLastError()));
      if (stream_out) {  // d mu / d S of this sub-shard are final: copy them out while the next runs
        const int64_t q = e->cfg.q, n = e->cfg.n_local;
        const int64_t ldm = e->g_mu.ld ? e->g_mu.ld : n, lds = e->g_s.ld ? e->g_s.ld : n;
        CUDA_OK(cudaEventRecord(e->ev_out[j], ctx->stream));
        CUDA_OK(cudaStreamWaitEvent(e->copy, e->ev_out[j], 0));
        CUDA_OK(cudaMemcpy2DAsync(e->g_mu.data + sub.n0, sizeof(double) * ldm, e->dmu.get<double>() + sub.n0,
                                    sizeof(double) * n, sizeof(double) * sub.n, q, cudaMemcpyDeviceToHost, e->copy));
        CUDA_OK(cudaMemcpy2DAsync(e->g_s.data + sub.n0, sizeof(double) * lds, e->ds.get<double>() + sub.n0,
                                    sizeof(double) * n, sizeof(double) * sub.n, q, cudaMemcpyDeviceToHost, e->copy));
      }
    }
    if (stream_out) {  // the read-backs join the stream (a captured graph needs every fork joined)
      if (!e->ev_copy_done) CUDA_OK(cudaEventCreateWithFlags(&e->ev_copy_done, cudaEventDisableTiming));
      CUDA_OK(cudaEventRecord(e->ev_copy_done, e->copy));
      CUDA_OK(cudaStreamWaitEvent(ctx->stream, e->ev_copy_done, 0));
    }
    if (k > 1) {
      if (red_side) {
        CUDA_OK(cudaEventRecord(e->ev_red[1], e->side2));
        CUDA_OK(cudaStreamWaitEvent(ctx->stream, e->ev_red[1], 0));
      }
      sum_parts_kernel<<<int(std::min<int64_t>((count + 255) / 256, 1024)), 256, 0, ctx->stream>>>(
          e->pgrads_sub.get<double>(), k, count, e->pgrads.get<double>());
      CUDA_OK(cudaGetLastError());
    }
  } else {
    join();
    CUDA_OK(cudaMemsetAsync(e->pgrads.p, 0, sizeof(double) * count, ctx->stream));
  }
  CUDA_OK(record_event(e->ev[3], ctx->stream));
  if (e->dev_coord) {  // d Kmm, Phi G for the assembly, behind the gradient kernels on the stream
    if (!e->split && dc_deferred(e->dc, ctx->stream)) throw CudaError("coordinator launch");
    return;
  }
  // host-only adjoints, overlapping the kernels just enqueued
  coord::complete_adjoints(e->res, e->st, e->cfg.n_global, e->cfg.d, e->beta);
}

// Device-coordinator finish: assembly kernel, then ONE read-back of the scalars, the gradient vector,
// the validation flag and the statistics; the reference's exceptions are raised from them in the
// reference's order (data validation, contract checks, factorizations, non-finite bound).
// stream part: the assembly kernel and the read-back copies (captured into the evaluation's graph)
void engine_finish_enqueue(sgpx_engine* e) {
  sgpx_ctx* ctx = e->ctx;
  if (e->split_join) {  // bound-only evaluation: the side stream's bound terms
    CUDA_OK(cudaStreamWaitEvent(ctx->stream, e->ev_split[1], 0));
    e->split_join = false;
  }
  const int64_t m = e->cfg.m, q = e->cfg.q, d = e->cfg.d;
  const DcArgs& dc = e->dc;
  if (e->with_grads && dc_finish(dc, e->pgrads.get<double>(), ctx->stream)) throw CudaError("coordinator launch");
  const int64_t nsc = kScCount, nres = 2 + q + m * q, nst = sgpx_packed_stats_count(m, d);
  e->h_dc.ensure(sizeof(double) * (nsc + nres + nst) + 16);
  double* h = e->h_dc.get<double>();
  CUDA_OK(cudaMemcpyAsync(h, dc.sc, sizeof(double) * nsc, cudaMemcpyDeviceToHost, ctx->stream));
  if (e->with_grads)
    CUDA_OK(cudaMemcpyAsync(h + nsc, dc.result, sizeof(double) * nres, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OK(cudaMemcpyAsync(h + nsc + nres, e->pstats.p, sizeof(double) * nst, cudaMemcpyDeviceToHost, ctx->stream));
  int* herr = reinterpret_cast<int*>(h + nsc + nres + nst);
  CUDA_OK(cudaMemcpyAsync(herr, e->err.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
}

void engine_finish_device(sgpx_engine* e, sgpx_eval_result* out, bool enqueued = false) {
  sgpx_ctx* ctx = e->ctx;
  const int64_t m = e->cfg.m, q = e->cfg.q, d = e->cfg.d;
  if (!enqueued) engine_finish_enqueue(e);
  const int64_t nsc = kScCount, nres = 2 + q + m * q, nst = sgpx_packed_stats_count(m, d);
  double* h = e->h_dc.get<double>();
  int* herr = reinterpret_cast<int*>(h + nsc + nres + nst);
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
  if (e->copy) CUDA_OK(cudaStreamSynchronize(e->copy));  // streamed d mu / d S have landed
  check_err_flag(*herr);
  const int st = int(h[kScStatus]);
  if (st & kStGramFailed)
    throw NumericError("factor_gram: Gram matrix not factorizable even at jitter 1e-2 * variance (ill-conditioned "
                       "inducing inputs)");
  require(!(st & kStBadCount), "bound: stats n_count does not match N");
  require(!(st & kStBadStats), "bound: phi and yy must be non-negative");
  if (st & kStAFailed)
    throw NumericError("bound (Kmm + beta*Phi): Cholesky factorization failed after jitter escalation");
  if (st & kStNonFinite) throw NumericError("bound: non-finite value");
  const double* bd = h + kScBound;
  out->bound = sgpx_bound_breakdown{bd[0], bd[1], bd[2], bd[3], bd[4], bd[5], bd[6]};
  e->last_bound = bd[0];
  const coord::Stats stt = coord::unpack_stats(h + nsc + nres, m, d);
  out->phi = stt.phi;
  out->yy = stt.yy;
  out->n_count = int64_t(stt.n);
  if (out->psi_y) std::copy(stt.psi_y.v.begin(), stt.psi_y.v.end(), out->psi_y);
  if (out->phi_big) std::copy(stt.phi_big.v.begin(), stt.phi_big.v.end(), out->phi_big);
  out->jitter_factor_used = h[kScJitterFactor];
  out->has_grads = e->with_grads ? 1 : 0;
  float ms = 0.f;
  if (e->with_grads) {
    const double* g = h + nsc;
    out->d_variance = g[0];
    if (out->d_lengthscales) std::copy(g + 1, g + 1 + q, out->d_lengthscales);
    if (out->d_z) std::copy(g + 1 + q, g + 1 + q + m * q, out->d_z);
    out->d_beta = g[1 + q + m * q];
    cudaEventElapsedTime(&ms, e->ev[2], e->ev[3]);
    out->grad_pass_s = ms * 1e-3;
    ms = 0.f;
    if (e->in.n > 0) cudaEventElapsedTime(&ms, e->ev[6], e->ev[7]);
    out->bwd_kernel_s = ms * 1e-3;
    ms = 0.f;
    if (e->in.n > 0 && cudaEventElapsedTime(&ms, e->ev[10], e->ev[11]) != cudaSuccess) {
      cudaGetLastError();
      ms = 0.f;
    }
    out->psi2_bwd_kernel_s = ms * 1e-3;
  } else {
    out->d_variance = 0.0;
    out->d_beta = 0.0;
    out->grad_pass_s = 0.0;
    out->bwd_kernel_s = 0.0;
    out->psi2_bwd_kernel_s = 0.0;
  }
  ms = 0.f;
  cudaEventElapsedTime(&ms, e->ev_c[0], e->ev_c[1]);
  e->coord_s = ms * 1e-3;  // device time of the coordinator kernels
}

void engine_finish(sgpx_engine* e, sgpx_eval_result* out, bool enqueued = false) {
  require(out != nullptr, "engine: result pointer is null");
  require(e->coordinated, "engine: coordinate must precede finish");
  if (e->dev_coord) {
    engine_finish_device(e, out, enqueued);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e->ev[0], e->ev[1]);
    out->stats_pass_s = ms * 1e-3;
    ms = 0.f;
    if (e->in.n > 0) cudaEventElapsedTime(&ms, e->ev[4], e->ev[5]);
    out->fwd_kernel_s = ms * 1e-3;
    ms = 0.f;
    if (e->in.n > 0 && cudaEventElapsedTime(&ms, e->ev[8], e->ev[9]) != cudaSuccess) {
      cudaGetLastError();
      ms = 0.f;
    }
    out->psi2_fwd_kernel_s = ms * 1e-3;
    out->fwd_grid = e->gf.grid;
    out->bwd_grid = e->with_grads ? e->gb.grid : 0;
    out->coordinator_s = e->coord_s;
    out->precision_used = e->P.mode;
    out->z_spread = e->z_spread;
    return;
  }
  sgpx_ctx* ctx = e->ctx;
  const int64_t m = e->cfg.m, q = e->cfg.q, d = e->cfg.d;

  const coord::Stats st = coord::unpack_stats(e->h_stats.get<double>(), m, d);
  out->bound = sgpx_bound_breakdown{e->res.bd.total,     e->res.bd.log_det,   e->res.bd.data_fit, e->res.bd.quadratic,
                                    e->res.bd.trace_phi, e->res.bd.trace_kmm, e->res.bd.kl};
  e->last_bound = e->res.bd.total;
  out->phi = st.phi;
  out->yy = st.yy;
  out->n_count = int64_t(st.n);
  if (out->psi_y) std::copy(st.psi_y.v.begin(), st.psi_y.v.end(), out->psi_y);
  if (out->phi_big) std::copy(st.phi_big.v.begin(), st.phi_big.v.end(), out->phi_big);
  out->jitter_factor_used = e->res.gram.jitter_factor;
  out->has_grads = e->with_grads ? 1 : 0;
  float ms = 0.f;
  if (e->with_grads) {
    const int64_t count = sgpx_packed_grads_count(m, q);
    e->h_grads.ensure(sizeof(double) * count);
    CUDA_OK(cudaMemcpyAsync(e->h_grads.p, e->pgrads.p, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    if (e->copy) CUDA_OK(cudaStreamSynchronize(e->copy));  // streamed d mu / d S have landed
    const double* g = e->h_grads.get<double>();
    coord::complete_adjoints(e->res, e->st, e->cfg.n_global, e->cfg.d, e->beta);
    coord::KernGrads kg = coord::kern_grads_zz(e->z, e->kernel, e->res.adj.d_kmm);
    double tr = 0.0;
    for (int64_t i = 0; i < m; ++i) tr += e->res.adj.d_kmm(i, i);
    out->d_variance = g[0] + kg.d_variance + e->res.gram.jitter_factor * tr;
    if (out->d_lengthscales)
      for (int64_t j = 0; j < q; ++j) out->d_lengthscales[j] = g[1 + j] + kg.d_ls[j];
    if (out->d_z)
      for (int64_t i = 0; i < m * q; ++i) out->d_z[i] = g[1 + q + i] + kg.d_z.v[i];
    out->d_beta = e->res.adj.d_beta;
    cudaEventElapsedTime(&ms, e->ev[2], e->ev[3]);
    out->grad_pass_s = ms * 1e-3;
    ms = 0.f;
    if (e->in.n > 0) cudaEventElapsedTime(&ms, e->ev[6], e->ev[7]);
    out->bwd_kernel_s = ms * 1e-3;
    ms = 0.f;
    if (e->in.n > 0 && cudaEventElapsedTime(&ms, e->ev[10], e->ev[11]) != cudaSuccess) {
      cudaGetLastError();
      ms = 0.f;
    }
    out->psi2_bwd_kernel_s = ms * 1e-3;
  } else {
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    out->d_variance = 0.0;
    out->d_beta = 0.0;
    out->grad_pass_s = 0.0;
    out->bwd_kernel_s = 0.0;
    out->psi2_bwd_kernel_s = 0.0;
  }
  cudaEventElapsedTime(&ms, e->ev[0], e->ev[1]);
  out->stats_pass_s = ms * 1e-3;
  ms = 0.f;
  if (e->in.n > 0) cudaEventElapsedTime(&ms, e->ev[4], e->ev[5]);
  out->fwd_kernel_s = ms * 1e-3;
  ms = 0.f;
  if (e->in.n > 0 && cudaEventElapsedTime(&ms, e->ev[8], e->ev[9]) != cudaSuccess) {
    cudaGetLastError();
    ms = 0.f;
  }
  out->psi2_fwd_kernel_s = ms * 1e-3;
  out->fwd_grid = e->gf.grid;
  out->bwd_grid = e->with_grads ? e->gb.grid : 0;
  out->coordinator_s = e->coord_s;
  out->precision_used = e->P.mode;
  out->z_spread = e->z_spread;
}

}  // namespace
}  // namespace sgpx

extern "C" {

const char* sgpx_last_error(void) { return g_last_error.c_str(); }
int sgpx_abi_version(void) { return SGPX_ABI_VERSION; }

int sgpx_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int sgpx_ctx_create(int device, sgpx_ctx** out) {
  return guard([&] {
    require(out != nullptr, "ctx_create: out is null");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw CudaError("no CUDA device: the B200 psi-statistics engine has no CPU fallback");
    }
    require(device >= 0 && device < n, "ctx_create: device index out of range");
    CUDA_OK(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      throw CudaError("device " + std::string(prop.name) + " is not sm_100-class; libsgpx is built for sm_100a");
    auto c = std::make_unique<sgpx_ctx>();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    c->launches0 = launches_issued();
    *out = c.release();
  });
}

int sgpx_ctx_destroy(sgpx_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int sgpx_ctx_set_stream(sgpx_ctx* ctx, void* stream) {
  return guard([&] {
    require(ctx != nullptr, "ctx is null");
    CUDA_OK(cudaSetDevice(ctx->device));
    if (ctx->own_stream && ctx->stream) CUDA_OK(cudaStreamDestroy(ctx->stream));
    ctx->stream = static_cast<cudaStream_t>(stream);
    ctx->own_stream = false;
  });
}

int sgpx_ctx_synchronize(sgpx_ctx* ctx) {
  return guard([&] {
    require(ctx != nullptr, "ctx is null");
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
  });
}

int64_t sgpx_ctx_launch_count(const sgpx_ctx* ctx) { return ctx ? launches_issued() - ctx->launches0 : 0; }

int sgpx_ctx_set_precision(sgpx_ctx* ctx, int precision) {
  return guard([&] {
    require(ctx != nullptr, "ctx is null");
    require(precision == SGPX_PREC_AUTO || precision == SGPX_PREC_FAST || precision == SGPX_PREC_PRECISE ||
                precision == SGPX_PREC_DIRECT || precision == SGPX_PREC_SYRK,
            "unknown precision mode");
    ctx->precision = precision;
  });
}

int sgpx_ctx_last_precision(const sgpx_ctx* ctx, double* z_spread) {
  if (!ctx) return 0;
  if (z_spread) *z_spread = ctx->last_z_spread;
  return ctx->last_mode;
}

int64_t sgpx_packed_stats_count(int64_t m, int64_t d) { return 4 + m * (m + 1) / 2 + m * d; }
int64_t sgpx_packed_grads_count(int64_t m, int64_t q) { return 1 + q + m * q; }

// ---- sweep_stats (psi_stats.hpp:108-326) ------------------------------------
int sgpx_sweep_stats(sgpx_ctx* ctx, int expected, sgpx_cmat mu, sgpx_cmat s, sgpx_cmat y, sgpx_cmat z,
                     const sgpx_kernel_spec* kernel, const sgpx_tile_config* tiles, const sgpx_stats_adjoints* adj,
                     sgpx_sufficient_stats* stats, sgpx_stats_grads* grads) {
  return guard([&] {
    require(ctx != nullptr, "ctx is null");
    require(stats != nullptr, "stats output is null");
    coord::Kernel k = kernel_from(kernel);
    if (tiles) require(tiles->block_span >= 1 && tiles->thread_span >= 1, "TileConfig spans must be >= 1");
    check_view(mu, "mu");
    check_view(y, "y");
    check_view(z, "z");
    const int64_t n = mu.rows, q = mu.cols, m = z.rows, d = y.cols;
    require(z.cols == q, "stats sweep: Z column count mismatch");
    require(int64_t(k.ls.size()) == q, "stats sweep: kernel dimension mismatch");
    require(y.rows == n, "stats sweep: X/Y row counts differ");
    if (expected) {
      check_view(s, "s");
      require(s.rows == n && s.cols == q, "VariationalPosterior: mu and s shapes differ");
    }
    coord::Mat zm = mat_from(z);
    require(all_finite(zm), "stats sweep: non-finite data");
    coord::Mat dphi_big, dpsi;
    if (adj) {
      require(adj->d_psi_y.rows == m && adj->d_psi_y.cols == d, "stats adjoints: d_psi_y shape must be M x D");
      require(adj->d_phi_big.rows == m && adj->d_phi_big.cols == m, "stats adjoints: d_phi_big shape must be M x M");
      dphi_big = mat_from(adj->d_phi_big);
      dpsi = mat_from(adj->d_psi_y);
      double scale = 0.0, asym = 0.0;
      for (int64_t j = 0; j < m; ++j)
        for (int64_t i = 0; i < m; ++i) {
          scale = std::max(scale, std::fabs(dphi_big(i, j)));
          asym = std::max(asym, std::fabs(dphi_big(i, j) - dphi_big(j, i)));
        }
      require(asym <= 1e-10 * (1.0 + scale), "stats adjoints: d_phi_big must be symmetric");
    }
    CUDA_OK(cudaSetDevice(ctx->device));
    // Reference semantics: outputs fully overwritten (psi_stats.hpp:123-134).
    stats->phi = double(n) * k.variance;
    stats->n_count = n;
    stats->yy = 0.0;
    coord::Mat zero_psi(m, d), zero_phi(m, m);
    if (grads) {
      coord::Mat zq(m, q);
      mat_to(zq, grads->d_z);
      grads->d_variance = adj ? adj->d_phi * double(n) : 0.0;
      if (grads->d_lengthscales) std::fill(grads->d_lengthscales, grads->d_lengthscales + q, 0.0);
      if (expected) {
        coord::Mat nq(n, q);
        mat_to(nq, grads->d_mu);
        mat_to(nq, grads->d_s);
      }
    }
    if (n == 0 || m == 0) {
      mat_to(zero_psi, stats->psi_y);
      mat_to(zero_phi, stats->phi_big);
      return;
    }
    upload(ctx, ctx->mu, mu, false);
    if (expected) upload(ctx, ctx->s, s, false);
    upload(ctx, ctx->y, y, false);
    ShardInputs in;
    in.n = n;
    in.q = q;
    in.d = d;
    in.m = m;
    in.expected = expected != 0;
    in.mu = ctx->mu.get<double>();
    in.ld_mu = n;
    in.s = expected ? ctx->s.get<double>() : nullptr;
    in.ld_s = n;
    in.y = ctx->y.get<double>();
    in.ld_y = n;
    PsiConst P = make_const(ctx, in, k, zm, ctx->zc, ctx->z64, ctx->h_stage, ctx->precision);
    ctx->last_mode = P.mode;
    ctx->last_z_spread = psi_z_spread(P, zm.v.data(), zm.r);
    LaunchGeom g{};
    if (plan_forward(P, ctx->num_sms, &g)) throw CudaError("psi forward: launch planning failed");
    ctx->fpart.ensure(sizeof(double) * fwd_part_count(P.m, P.d) * std::max(1, g.grid));
    const int64_t count = sgpx_packed_stats_count(m, d);
    ctx->pstats.ensure(sizeof(double) * count);
    ctx->err.ensure(sizeof(int));
    CUDA_OK(cudaMemsetAsync(ctx->err.p, 0, sizeof(int), ctx->stream));
    if (psi_forward(P, ctx->fpart.get<double>(), ctx->pstats.get<double>(), ctx->err.get<int>(), ctx->num_sms,
                    ctx->stream, nullptr))
      throw CudaError(std::string("psi forward launch: ") + cudaGetErrorString(cudaGetLastError()));
    ctx->h_stats.ensure(sizeof(double) * count);
    ctx->h_err.ensure(sizeof(int));
    CUDA_OK(cudaMemcpyAsync(ctx->h_stats.p, ctx->pstats.p, sizeof(double) * count, cudaMemcpyDeviceToHost,
                              ctx->stream));
    CUDA_OK(cudaMemcpyAsync(ctx->h_err.p, ctx->err.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    check_err_flag(*ctx->h_err.get<int>());
    const coord::Stats st = coord::unpack_stats(ctx->h_stats.get<double>(), m, d);
    stats->yy = st.yy;
    mat_to(st.psi_y, stats->psi_y);
    mat_to(st.phi_big, stats->phi_big);
    if (!grads || !adj) return;

    stage_adjoints(P, dphi_big, dpsi, ctx->h_u, ctx->h_dpsi);
    upload_adjoints(P, ctx->h_u, ctx->h_dpsi, ctx->u, ctx->dpsi, ctx->u64, ctx->dpsi64, ctx->stream);
    ctx->dmu.ensure(sizeof(double) * n * q);
    ctx->ds.ensure(sizeof(double) * n * q);
    BwdConst B{};
    B.u = ctx->u.get<float>();
    B.dpsi = ctx->dpsi.get<float>();
    B.u64 = ctx->u64.get<double>();
    B.dpsi64 = ctx->dpsi64.get<double>();
    B.d_phi = adj->d_phi;
    B.add_kl = 0;
    B.write_local = expected ? 1 : 0;
    B.d_mu = ctx->dmu.get<double>();
    B.d_s = ctx->ds.get<double>();
    B.ld_g = n;
    B.fwd_rt = fwd_region(P, ctx->fpart.get<double>(), ctx->num_sms);
    if (plan_backward(P, ctx->num_sms, &g)) throw CudaError("psi backward: launch planning failed");
    ctx->bpart.ensure(sizeof(double) * bwd_part_count(P.m, P.q) * std::max(1, g.grid));
    const int64_t gcount = sgpx_packed_grads_count(m, q);
    ctx->pgrads.ensure(sizeof(double) * gcount);
    if (psi_backward(P, B, ctx->bpart.get<double>(), ctx->pgrads.get<double>(), ctx->num_sms, ctx->stream, nullptr))
      throw CudaError(std::string("psi backward launch: ") + cudaGetErrorString(cudaGetLastError()));
    ctx->h_grads.ensure(sizeof(double) * gcount);
    CUDA_OK(cudaMemcpyAsync(ctx->h_grads.p, ctx->pgrads.p, sizeof(double) * gcount, cudaMemcpyDeviceToHost,
                              ctx->stream));
    if (expected) {
      const int64_t ldm = grads->d_mu.ld ? grads->d_mu.ld : grads->d_mu.rows;
      const int64_t lds = grads->d_s.ld ? grads->d_s.ld : grads->d_s.rows;
      require(grads->d_mu.data && grads->d_s.data, "stats grads: d_mu / d_s outputs are null");
      CUDA_OK(cudaMemcpy2DAsync(grads->d_mu.data, sizeof(double) * ldm, ctx->dmu.p, sizeof(double) * n,
                                  sizeof(double) * n, q, cudaMemcpyDeviceToHost, ctx->stream));
      CUDA_OK(cudaMemcpy2DAsync(grads->d_s.data, sizeof(double) * lds, ctx->ds.p, sizeof(double) * n,
                                  sizeof(double) * n, q, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    const double* gg = ctx->h_grads.get<double>();
    grads->d_variance = gg[0];
    if (grads->d_lengthscales)
      for (int64_t j = 0; j < q; ++j) grads->d_lengthscales[j] = gg[1 + j];
    coord::Mat dz(m, q);
    std::copy(gg + 1 + q, gg + 1 + q + m * q, dz.v.begin());
    mat_to(dz, grads->d_z);
  });
}

int sgpx_psi1_expected(sgpx_ctx* ctx, sgpx_cmat mu, sgpx_cmat s, sgpx_cmat z, const sgpx_kernel_spec* kernel,
                       sgpx_mmat out) {
  return guard([&] {
    require(ctx != nullptr, "ctx is null");
    coord::Kernel k = kernel_from(kernel);
    check_view(mu, "mu");
    check_view(s, "s");
    check_view(z, "z");
    const int64_t n = mu.rows, q = mu.cols, m = z.rows;
    require(s.rows == n && s.cols == q, "VariationalPosterior: mu and s shapes differ");
    require(z.cols == q, "psi1_expected: Z column count mismatch");
    require(int64_t(k.ls.size()) == q, "psi1_expected: kernel dimension mismatch");
    require(out.rows == n && out.cols == m && (n * m == 0 || out.data), "psi1_expected: output must be N x M");
    coord::Mat zm = mat_from(z);
    CUDA_OK(cudaSetDevice(ctx->device));
    if (n * m == 0) return;
    upload(ctx, ctx->mu, mu, false);
    upload(ctx, ctx->s, s, false);
    ShardInputs in;
    in.n = n;
    in.q = q;
    in.m = m;
    in.d = 0;
    in.expected = true;
    in.mu = ctx->mu.get<double>();
    in.ld_mu = n;
    in.s = ctx->s.get<double>();
    in.ld_s = n;
    PsiConst P = make_const(ctx, in, k, zm, ctx->zc, ctx->z64, ctx->h_stage, SGPX_PREC_DIRECT);
    ctx->out.ensure(sizeof(double) * n * m);
    // validation (VariationalPosterior::validate, psi_stats.hpp:20-25) via the forward err flag is
    // not run here; check on the host copy instead.
    {
      const int64_t ldm = mu.ld ? mu.ld : n, lds = s.ld ? s.ld : n;
      for (int64_t j = 0; j < q; ++j)
        for (int64_t i = 0; i < n; ++i) {
          require(std::isfinite(mu.data[i + j * ldm]) && std::isfinite(s.data[i + j * lds]),
                  "VariationalPosterior: non-finite entries");
          require(s.data[i + j * lds] > 0.0, "VariationalPosterior: variances must be positive");
        }
    }
    if (psi1_matrix(P, ctx->out.get<double>(), n, ctx->stream))
      throw CudaError(std::string("psi1 launch: ") + cudaGetErrorString(cudaGetLastError()));
    const int64_t ldo = out.ld ? out.ld : n;
    CUDA_OK(cudaMemcpy2DAsync(out.data, sizeof(double) * ldo, ctx->out.p, sizeof(double) * n, sizeof(double) * n, m,
                                cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
  });
}

int sgpx_psi0_expected(sgpx_cmat mu, sgpx_cmat s, const sgpx_kernel_spec* kernel, double* out) {
  return guard([&] {
    coord::Kernel k = kernel_from(kernel);
    check_view(mu, "mu");
    check_view(s, "s");
    require(mu.rows == s.rows && mu.cols == s.cols, "VariationalPosterior: mu and s shapes differ");
    require(out != nullptr, "psi0_expected: out is null");
    *out = double(mu.rows) * k.variance;
  });
}

// ---- coordinator (host) -------------------------------------------------------
int sgpx_coordinate_host(int kind, int64_t n, int64_t d, int64_t m, const double* packed_stats, sgpx_cmat z,
                         const sgpx_kernel_spec* kernel, double beta, double jitter_factor, sgpx_bound_breakdown* bd,
                         double* adj_scalars, double* d_psi_y, double* d_phi_big, double* d_kmm) {
  return guard([&] {
    require(packed_stats && bd, "coordinate: null input/output");
    coord::Kernel k = kernel_from(kernel);
    require(z.rows == m, "coordinate: Z must have M rows");
    coord::Mat zm = mat_from(z);
    const coord::Stats st = coord::unpack_stats(packed_stats, m, d);
    const bool want = adj_scalars != nullptr;
    coord::Result r = coord::coordinate(kind == 1, n, d, st, zm, k, beta, jitter_factor, want);
    *bd = sgpx_bound_breakdown{r.bd.total, r.bd.log_det, r.bd.data_fit, r.bd.quadratic, r.bd.trace_phi, r.bd.trace_kmm,
                               r.bd.kl};
    if (want) {
      adj_scalars[0] = r.adj.d_phi;
      adj_scalars[1] = r.adj.d_beta;
      adj_scalars[2] = r.gram.jitter_factor;
      if (d_psi_y) std::copy(r.adj.d_psi_y.v.begin(), r.adj.d_psi_y.v.end(), d_psi_y);
      if (d_phi_big) std::copy(r.adj.d_phi_big.v.begin(), r.adj.d_phi_big.v.end(), d_phi_big);
      if (d_kmm) std::copy(r.adj.d_kmm.v.begin(), r.adj.d_kmm.v.end(), d_kmm);
    }
  });
}

int sgpx_finish_host(int64_t m, int64_t q, const double* packed_grads, sgpx_cmat z, const sgpx_kernel_spec* kernel,
                     const double* d_kmm, double jitter_factor, double* d_z, double* d_variance, double* d_ls) {
  return guard([&] {
    require(packed_grads && d_kmm && d_z && d_variance && d_ls, "finish: null input/output");
    coord::Kernel k = kernel_from(kernel);
    coord::Mat zm = mat_from(z);
    coord::Mat dk(m, m);
    std::copy(d_kmm, d_kmm + m * m, dk.v.begin());
    coord::KernGrads kg = coord::kern_grads_zz(zm, k, dk);
    double tr = 0.0;
    for (int64_t i = 0; i < m; ++i) tr += dk(i, i);
    *d_variance = packed_grads[0] + kg.d_variance + jitter_factor * tr;
    for (int64_t j = 0; j < q; ++j) d_ls[j] = packed_grads[1 + j] + kg.d_ls[j];
    for (int64_t i = 0; i < m * q; ++i) d_z[i] = packed_grads[1 + q + i] + kg.d_z.v[i];
  });
}

// ---- engine -------------------------------------------------------------------
int sgpx_engine_create(sgpx_ctx* ctx, const sgpx_engine_config* cfg, sgpx_engine** out) {
  return guard([&] {
    require(ctx && cfg && out, "engine_create: null argument");
    require(cfg->kind == 0 || cfg->kind == 1, "engine_create: kind must be 0 (regression) or 1 (latent)");
    require(cfg->n_local >= 0 && cfg->row_begin >= 0 && cfg->row_begin + cfg->n_local <= cfg->n_global,
            "engine_create: shard rows outside [0, N)");
    require(cfg->q >= 1 && cfg->q <= kMaxQ, "engine_create: Q must be in [1, 64]");
    require(cfg->precision == SGPX_PREC_AUTO || cfg->precision == SGPX_PREC_FAST ||
                cfg->precision == SGPX_PREC_PRECISE || cfg->precision == SGPX_PREC_DIRECT ||
                cfg->precision == SGPX_PREC_SYRK,
            "engine_create: unknown precision mode");
    require(cfg->m >= 1 && cfg->d >= 1, "engine_create: need M >= 1 and D >= 1");
    require(cfg->jitter_factor >= 0.0, "factor_gram: jitter factor must be non-negative");
    CUDA_OK(cudaSetDevice(ctx->device));
    auto e = std::make_unique<sgpx_engine>();
    e->ctx = ctx;
    e->cfg = *cfg;
    e->latent = cfg->kind == 1;
    for (auto& ev : e->ev) CUDA_OK(cudaEventCreate(&ev));
    for (auto& ev : e->ev_c) CUDA_OK(cudaEventCreate(&ev));
    // device coordinator by default: stream-ordered (no host round trip between the passes), split so
    // that only the factorisation and G = A^-1 Psi sit between the passes (C3: 5.78 vs 6.08 ms per
    // evaluation, end to end 7.98 vs 8.23 ms; profiles/r02/coord_split_ab.txt); the host coordinator
    // (SGPX_DEVICE_COORD=0) remains for A/B
    e->dev_coord = true;
    if (const char* dc = getenv("SGPX_DEVICE_COORD")) e->dev_coord = atoi(dc) != 0;  // A/B
    if (const char* sp = getenv("SGPX_COORD_SPLIT")) e->coord_split = atoi(sp) != 0;  // A/B
    if (const char* gr = getenv("SGPX_GRAPH")) e->use_graph = atoi(gr) != 0;       // A/B: per-call launches
    *out = e.release();
  });
}

int sgpx_engine_destroy(sgpx_engine* eng) {
  return guard([&] {
    if (!eng) return;
    cudaSetDevice(eng->ctx->device);
    delete eng;
  });
}

int sgpx_engine_set_data(sgpx_engine* e, sgpx_cmat x_or_mu, sgpx_cmat s, sgpx_cmat y, int on_device) {
  return guard([&] {
    require(e != nullptr, "engine is null");
    const int64_t n = e->cfg.n_local, q = e->cfg.q, d = e->cfg.d;
    check_view(x_or_mu, "x_or_mu");
    check_view(y, "y");
    require(y.rows == n && y.cols == d, "worker: Y must be n_local x D");
    require(x_or_mu.rows == n && x_or_mu.cols == q, "worker: X/mu must be n_local x Q");
    if (e->latent) {
      check_view(s, "s");
      require(s.rows == n && s.cols == q, "worker: local parameter row mismatch");
    }
    CUDA_OK(cudaSetDevice(e->ctx->device));
    ShardInputs& in = e->in;
    in.n = n;
    in.q = q;
    in.d = d;
    in.m = e->cfg.m;
    in.expected = e->latent;
    if (on_device) {  // adopt (the caller keeps the device buffers alive)
      in.mu = x_or_mu.data;
      in.ld_mu = x_or_mu.ld ? x_or_mu.ld : n;
      in.y = y.data;
      in.ld_y = y.ld ? y.ld : n;
      in.s = e->latent ? s.data : nullptr;
      in.ld_s = e->latent ? (s.ld ? s.ld : n) : n;
    } else {
      upload(e->ctx, e->own_x, x_or_mu, false);
      upload(e->ctx, e->own_y, y, false);
      in.mu = e->own_x.get<double>();
      in.ld_mu = n;
      in.y = e->own_y.get<double>();
      in.ld_y = n;
      if (e->latent) {
        upload(e->ctx, e->own_s, s, false);
        in.s = e->own_s.get<double>();
      }
      in.ld_s = n;
    }
    e->has_data = true;
    if (e->uploads_enqueued) {  // an earlier broadcast's copies must not land on top of these rows
      CUDA_OK(cudaStreamSynchronize(e->copy));
      e->uploads_enqueued = false;
    }
    e->pending_upload = false;  // rows set here replace any host views of an earlier broadcast
    if (e->has_params) {
      e->P.mu = in.mu;
      e->P.ld_mu = in.ld_mu;
      e->P.s = in.s;
      e->P.ld_s = in.ld_s;
      e->P.y = in.y;
      e->P.ld_y = in.ld_y;
    }
  });
}

int sgpx_engine_broadcast(sgpx_engine* e, const sgpx_kernel_spec* kernel, double beta, sgpx_cmat z, sgpx_cmat mu,
                          sgpx_cmat s, int on_device) {
  return guard([&] {
    require(e != nullptr, "engine is null");
    coord::Kernel k = kernel_from(kernel);
    require(int64_t(k.ls.size()) == e->cfg.q, "broadcast: kernel dimension mismatch");
    check_view(z, "z");
    require(z.rows == e->cfg.m && z.cols == e->cfg.q, "broadcast: Z must be M x Q");
    require(std::isfinite(beta) && beta > 0.0, "noise precision beta must be positive");
    require(e->has_data, "broadcast: set_data (the Engine's shard rows) must come first");
    CUDA_OK(cudaSetDevice(e->ctx->device));
    coord::Mat zm = mat_from(z);
    require(all_finite(zm), "stats sweep: non-finite data");
    if (e->latent && mu.data) {
      require(e->has_data, "broadcast: set_data must precede a local-parameter broadcast");
      check_view(mu, "mu");
      check_view(s, "s");
      require(mu.rows == e->cfg.n_local && s.rows == e->cfg.n_local && mu.cols == e->cfg.q && s.cols == e->cfg.q,
              "broadcast: local parameter row mismatch");
      if (on_device) {
        e->pending_upload = false;
        e->in.mu = mu.data;
        e->in.ld_mu = mu.ld ? mu.ld : e->cfg.n_local;
        e->in.s = s.data;
        e->in.ld_s = s.ld ? s.ld : e->cfg.n_local;
      } else {  // deferred: the stats pass streams the rows in sub-shards (overlapped with its kernels)
        const size_t bytes = sizeof(double) * std::max<int64_t>(1, e->cfg.n_local * e->cfg.q);
        e->own_x.ensure(bytes);
        e->own_s.ensure(bytes);
        e->h_mu = mu;
        e->h_s = s;
        if (e->uploads_enqueued) CUDA_OK(cudaStreamSynchronize(e->copy));  // an unconsumed earlier broadcast
        e->uploads_enqueued = false;
        e->pending_upload = e->cfg.n_local * e->cfg.q > 0;
        e->in.mu = e->own_x.get<double>();
        e->in.ld_mu = e->cfg.n_local;
        e->in.s = e->own_s.get<double>();
        e->in.ld_s = e->cfg.n_local;
      }
    }
    e->kernel = k;
    e->z = zm;
    e->beta = beta;
    e->P = make_const(e->ctx, e->in, k, zm, e->zc, e->z64, e->h_stage, e->cfg.precision);
    e->z_spread = psi_z_spread(e->P, zm.v.data(), zm.r);
    e->kernel_ls = k.ls;
    e->dc_ready = false;
    if (e->dev_coord) dc_setup(e);  // per-broadcast half of the coordinator (Kmm, its factor, inverse)
    e->has_params = true;
    e->coordinated = false;
    if (e->pending_upload && !(e->use_graph && e->dev_coord && e->ctx->stream != nullptr && is_pinned(mu.data) &&
                               is_pinned(s.data))) {
      // host mu / S: the transfer starts now, under the caller's work until evaluate (after the Z upload
      // above: copies in one direction share a copy engine, so a small copy queued behind these would wait
      // for all of them); the stats pass re-plans the same sub-shards with this broadcast's constants
      plan_subs(e);
      enqueue_uploads(e);
    }
  });
}

int sgpx_engine_stats_pass(sgpx_engine* e, double** packed_dev, int64_t* count) {
  return guard([&] {
    require(e != nullptr, "engine is null");
    CUDA_OK(cudaSetDevice(e->ctx->device));
    engine_stats_pass(e);
    if (packed_dev) *packed_dev = e->pstats.get<double>();
    if (count) *count = sgpx_packed_stats_count(e->cfg.m, e->cfg.d);
  });
}

int sgpx_engine_coordinate(sgpx_engine* e, int with_grads) {
  return guard([&] {
    require(e != nullptr, "engine is null");
    CUDA_OK(cudaSetDevice(e->ctx->device));
    engine_coordinate(e, with_grads != 0);
  });
}

int sgpx_engine_grad_pass(sgpx_engine* e, double** packed_dev, int64_t* count) {
  return guard([&] {
    require(e != nullptr, "engine is null");
    CUDA_OK(cudaSetDevice(e->ctx->device));
    engine_grad_pass(e);
    if (packed_dev) *packed_dev = e->pgrads.get<double>();
    if (count) *count = sgpx_packed_grads_count(e->cfg.m, e->cfg.q);
  });
}

int sgpx_engine_finish(sgpx_engine* e, sgpx_eval_result* out) {
  return guard([&] {
    require(e != nullptr, "engine is null");
    CUDA_OK(cudaSetDevice(e->ctx->device));
    engine_finish(e, out);
  });
}

int sgpx_engine_evaluate(sgpx_engine* e, int with_grads, sgpx_eval_result* out) {
  return guard([&] {
    require(e != nullptr && out != nullptr, "engine/result is null");
    require(e->cfg.n_local == e->cfg.n_global, "engine_evaluate is the single-rank pipeline; use the phases");
    CUDA_OK(cudaSetDevice(e->ctx->device));
    const auto t0 = std::chrono::steady_clock::now();
    // graph replay: device-resident rows (no host streaming) and the device coordinator
    // (the legacy default stream cannot be captured)
    // (the host-buffer path too: the sub-shard uploads and read-backs are captured as copy nodes, the
    // host views and output buffers are part of the key)
    // (copies from pageable host memory cannot be captured: the host-buffer path is replayed only when
    // every host view is page-locked)
    const bool host_pinned = (!e->pending_upload || (is_pinned(e->h_mu.data) && is_pinned(e->h_s.data))) &&
                             (!(e->has_gout && e->latent) || (is_pinned(e->g_mu.data) && is_pinned(e->g_s.data)));
    const bool graphable = e->use_graph && e->dev_coord && !e->uploads_enqueued && host_pinned && e->in.n > 0 &&
                           e->has_data && e->has_params && e->ctx->stream != nullptr;
    if (graphable) {
      const bool host_io = e->pending_upload || (e->has_gout && e->latent);
      std::vector<unsigned char> key(sizeof(PsiConst) + sizeof(DcArgs) + 4 * sizeof(int) + 4 * sizeof(sgpx_cmat));
      unsigned char* p = key.data();
      std::memcpy(p, &e->P, sizeof(PsiConst));
      p += sizeof(PsiConst);
      std::memcpy(p, &e->dc, sizeof(DcArgs));
      p += sizeof(DcArgs);
      const int flags[4] = {with_grads ? 1 : 0, e->ctx->device,
                            (e->pending_upload ? 1 : 0) | (e->pre_needed ? 2 : 0) | (e->pre_pending ? 4 : 0),
                            (e->has_gout && e->latent) ? 1 : 0};
      std::memcpy(p, flags, sizeof(flags));
      p += sizeof(flags);
      const sgpx_cmat views[4] = {e->pending_upload ? e->h_mu : sgpx_cmat{}, e->pending_upload ? e->h_s : sgpx_cmat{},
                                  host_io ? sgpx_cmat{e->g_mu.data, e->g_mu.rows, e->g_mu.cols, e->g_mu.ld} : sgpx_cmat{},
                                  host_io ? sgpx_cmat{e->g_s.data, e->g_s.rows, e->g_s.cols, e->g_s.ld} : sgpx_cmat{}};
      std::memcpy(p, views, sizeof(views));
      cudaStream_t st = e->ctx->stream;
      if (!e->graph || key != e->graph_key) {
        if (e->graph) {
          cudaGraphExecDestroy(e->graph);
          e->graph = nullptr;
        }
        CUDA_OK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        const int64_t l0 = launches_issued();
        cudaGraph_t g = nullptr;
        try {
          engine_stats_pass(e);
          engine_coordinate(e, with_grads != 0);
          if (with_grads) engine_grad_pass(e);
          engine_finish_enqueue(e);
        } catch (...) {
          cudaStreamEndCapture(st, &g);
          if (g) cudaGraphDestroy(g);
          cudaGetLastError();
          throw;
        }
        CUDA_OK(cudaStreamEndCapture(st, &g));
        e->graph_launches = launches_issued() - l0;
        launches_add(-e->graph_launches);  // counted when the graph runs
        const cudaError_t ie = cudaGraphInstantiate(&e->graph, g, 0);
        cudaGraphDestroy(g);
        CUDA_OK(ie);
        e->graph_key = key;
      } else {
        e->with_grads = with_grads != 0;
        e->coordinated = true;
        e->pending_upload = false;  // (what the captured passes do on the host)
        e->pre_needed = e->pre_pending = false;
      }
      CUDA_OK(cudaGraphLaunch(e->graph, st));
      launches_add(e->graph_launches);
      engine_finish(e, out, true);
    } else {
      engine_stats_pass(e);
      engine_coordinate(e, with_grads != 0);
      if (with_grads) engine_grad_pass(e);
      engine_finish(e, out);
    }
    out->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// predict_from_cache (model.hpp:197-217) on the factors of the engine's last evaluation at the current
// parameters (the reference's finalize(): an evaluation after the last broadcast).
int sgpx_engine_predict(sgpx_engine* e, sgpx_cmat x_star, int observation, sgpx_mmat mean, sgpx_mmat var,
                        double* cached_bound) {
  return guard([&] {
    require(e != nullptr, "engine is null");
    require(e->coordinated && e->has_params, "predict() before fit()/finalize()");
    if (!e->dev_coord) {  // host-coordinated engine: rebuild the factors on the device from the last statistics
      CUDA_OK(cudaSetDevice(e->ctx->device));
      if (!e->dc_ready) dc_setup(e);
      dc_launch_prefactor(e);
      dc_join_prefactor(e);
      e->u.ensure(sizeof(float) * e->P.mv * e->P.mv);
      e->dpsi.ensure(sizeof(float) * std::max(1, e->P.d) * e->P.mv);
      e->u64.ensure(sizeof(double) * e->P.mv * e->P.mv);
      e->dpsi64.ensure(sizeof(double) * std::max(1, e->P.d) * e->P.mv);
      e->dc.packed = e->pstats.get<double>();
      if (dc_bound(e->dc, e->u.get<float>(), e->dpsi.get<float>(), e->u64.get<double>(), e->dpsi64.get<double>(),
                   e->ctx->stream))
        throw CudaError("coordinator launch");
    }
    check_view(x_star, "x_star");
    require(x_star.cols == e->cfg.q, "predict: X* column mismatch");
    const int64_t t = x_star.rows, d = e->cfg.d;
    require(mean.rows == t && mean.cols == d && var.rows == t && var.cols == d, "predict: outputs must be T x D");
    if (cached_bound) *cached_bound = e->last_bound;
    if (t == 0) return;
    CUDA_OK(cudaSetDevice(e->ctx->device));
    sgpx_ctx* ctx = e->ctx;
    const int64_t q = e->cfg.q, m = e->cfg.m;
    ctx->out.ensure(sizeof(double) * (t * q + 2 * t * d + dc_predict_doubles(t, int(m), int(q), int(d))));
    double* xs = ctx->out.get<double>();
    double* dmean = xs + t * q;
    double* dvar = dmean + t * d;
    double* work = dvar + t * d;
    CUDA_OK(cudaMemcpy2DAsync(xs, sizeof(double) * t, x_star.data, sizeof(double) * (x_star.ld ? x_star.ld : t),
                                sizeof(double) * t, q, cudaMemcpyHostToDevice, ctx->stream));
    if (dc_predict(e->dc, xs, t, observation ? 1 : 0, work, dmean, dvar, ctx->stream)) throw CudaError("predict launch");
    CUDA_OK(cudaMemcpy2DAsync(mean.data, sizeof(double) * (mean.ld ? mean.ld : t), dmean, sizeof(double) * t,
                                sizeof(double) * t, d, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(cudaMemcpy2DAsync(var.data, sizeof(double) * (var.ld ? var.ld : t), dvar, sizeof(double) * t,
                                sizeof(double) * t, d, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
  });
}

int sgpx_engine_set_local_grads_out(sgpx_engine* e, sgpx_mmat d_mu, sgpx_mmat d_s) {
  return guard([&] {
    require(e != nullptr, "engine is null");
    require(e->latent, "regression engines hold no local gradients");
    if (d_mu.data == nullptr && d_s.data == nullptr) {
      e->has_gout = false;
      return;
    }
    const int64_t n = e->cfg.n_local, q = e->cfg.q;
    require(d_mu.rows == n && d_mu.cols == q && d_s.rows == n && d_s.cols == q, "local grads must be n_local x Q");
    require(d_mu.data && d_s.data, "local grads out: null data");
    e->g_mu = d_mu;
    e->g_s = d_s;
    e->has_gout = true;
  });
}

int sgpx_engine_local_grads_device(sgpx_engine* e, double** d_mu, double** d_s) {
  return guard([&] {
    require(e != nullptr && d_mu && d_s, "null argument");
    require(e->latent, "regression engines hold no local gradients");
    *d_mu = e->dmu.get<double>();
    *d_s = e->ds.get<double>();
  });
}

int sgpx_engine_copy_local_grads(sgpx_engine* e, sgpx_mmat d_mu, sgpx_mmat d_s) {
  return guard([&] {
    require(e != nullptr, "engine is null");
    require(e->latent, "regression engines hold no local gradients");
    const int64_t n = e->cfg.n_local, q = e->cfg.q;
    require(d_mu.rows == n && d_mu.cols == q && d_s.rows == n && d_s.cols == q, "local grads must be n_local x Q");
    CUDA_OK(cudaSetDevice(e->ctx->device));
    CUDA_OK(cudaMemcpy2DAsync(d_mu.data, sizeof(double) * (d_mu.ld ? d_mu.ld : n), e->dmu.p, sizeof(double) * n,
                                sizeof(double) * n, q, cudaMemcpyDeviceToHost, e->ctx->stream));
    CUDA_OK(cudaMemcpy2DAsync(d_s.data, sizeof(double) * (d_s.ld ? d_s.ld : n), e->ds.p, sizeof(double) * n,
                                sizeof(double) * n, q, cudaMemcpyDeviceToHost, e->ctx->stream));
    CUDA_OK(cudaStreamSynchronize(e->ctx->stream));
  });
}

// ---- seeded inputs and binary matrices (common.hpp:45-97, model.hpp:420-429, io.hpp:114-153) ----
int sgpx_rng_normal_matrix(sgpx_ctx* ctx, uint64_t seed, int64_t rows, int64_t cols, sgpx_mmat out, int on_device) {
  return guard([&] {
    require(ctx != nullptr, "ctx is null");
    require(rows >= 0 && cols >= 0 && out.rows == rows && out.cols == cols, "rng: output must be rows x cols");
    require(rows * cols == 0 || out.data != nullptr, "rng: null output");
    const int64_t ld = out.ld ? out.ld : rows;
    require(ld >= rows, "rng: leading dimension smaller than rows");
    if (rows * cols == 0) return;
    CUDA_OK(cudaSetDevice(ctx->device));
    if (on_device) {
      if (rng_normal_device(seed, rows, cols, out.data, ld, ctx->stream)) throw CudaError("rng launch failed");
      CUDA_OK(cudaStreamSynchronize(ctx->stream));
      return;
    }
    ctx->out.ensure(sizeof(double) * rows * cols);
    if (rng_normal_device(seed, rows, cols, ctx->out.get<double>(), rows, ctx->stream))
      throw CudaError("rng launch failed");
    CUDA_OK(cudaMemcpy2DAsync(out.data, sizeof(double) * ld, ctx->out.p, sizeof(double) * rows, sizeof(double) * rows,
                                cols, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
  });
}

int sgpx_rng_choose_rows(uint64_t seed, int64_t n, int64_t m, int64_t* idx) {
  return guard([&] {
    require(m >= 1 && m <= n, "init_gplvm: need 1 <= M <= N");
    require(idx != nullptr, "rng: null output");
    rng_choose_rows(seed, n, m, idx);
  });
}

int sgpx_io_matrix_shape(const char* base, int64_t* rows, int64_t* cols) {
  return guard([&] {
    require(base && rows && cols, "io: null argument");
    io_read_shape(base, rows, cols);
  });
}

int sgpx_io_read_matrix(const char* base, sgpx_mmat out) {
  return guard([&] {
    require(base != nullptr, "io: null path");
    int64_t r = 0, c = 0;
    io_read_shape(base, &r, &c);
    require(out.rows == r && out.cols == c && (r * c == 0 || out.data), "io: output shape differs from the file");
    io_read_host(base, out.data, out.ld ? out.ld : r);
  });
}

int sgpx_io_write_matrix(const char* base, sgpx_cmat m) {
  return guard([&] {
    require(base != nullptr, "io: null path");
    check_view(m, "matrix");
    io_write_host(base, m.data, m.rows, m.cols, m.ld ? m.ld : m.rows);
  });
}

int sgpx_io_load_matrix_device(sgpx_ctx* ctx, const char* base, sgpx_mmat dev_out) {
  return guard([&] {
    require(ctx && base, "io: null argument");
    int64_t r = 0, c = 0;
    io_read_shape(base, &r, &c);
    require(dev_out.rows == r && dev_out.cols == c && (r * c == 0 || dev_out.data),
            "io: output shape differs from the file");
    CUDA_OK(cudaSetDevice(ctx->device));
    io_load_device(base, dev_out.data, dev_out.ld ? dev_out.ld : r, ctx->stream);
  });
}

// ---- multi-GPU engine: Engine(workers) of parallel.hpp:326-479 inside one process -----------------
// Shards = make_partition(N, workers) (parallel.hpp:28-41), shard i on devices[i] with its own
// context (stream).  Per evaluation: every shard's statistics pass -> exchange #1 -> the coordinator
// on every shard (redundant, no broadcast) -> every shard's gradient pass -> exchange #2 -> assembly.
// An exchange sums the packed fp64 buffers: shards that share a device are folded into the first of
// them (ascending shard order, stream events order the cross-stream reads), then one ncclAllReduce
// (sum, fp64) runs among the first shards of the distinct devices over NVLink / NVSwitch (one NCCL
// communicator per device from ncclCommInitAll), and the result is copied back to the device's other
// shards.  NCCL is opened at run time (dlopen), so the library loads on hosts without it.
}  // extern "C"

#include <dlfcn.h>

namespace sgpx {
namespace {

typedef int (*nccl_init_all_t)(void** comms, int ndev, const int* devlist);
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_group_t)();
typedef int (*nccl_destroy_t)(void*);
typedef const char* (*nccl_err_t)(int);

struct NcclApi {
  void* h = nullptr;
  nccl_init_all_t init_all = nullptr;
  nccl_allreduce_t allreduce = nullptr;
  nccl_group_t group_start = nullptr, group_end = nullptr;
  nccl_destroy_t destroy = nullptr;
  nccl_err_t err = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return a;
    a.init_all = reinterpret_cast<nccl_init_all_t>(dlsym(a.h, "ncclCommInitAll"));
    a.allreduce = reinterpret_cast<nccl_allreduce_t>(dlsym(a.h, "ncclAllReduce"));
    a.group_start = reinterpret_cast<nccl_group_t>(dlsym(a.h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<nccl_group_t>(dlsym(a.h, "ncclGroupEnd"));
    a.destroy = reinterpret_cast<nccl_destroy_t>(dlsym(a.h, "ncclCommDestroy"));
    a.err = reinterpret_cast<nccl_err_t>(dlsym(a.h, "ncclGetErrorString"));
    return a;
  }();
  return api;
}

void nccl_ok(int rc, const char* what) {
  if (rc != 0) {
    const NcclApi& a = nccl_api();
    throw NcclError(std::string(what) + ": " + (a.err ? a.err(rc) : "NCCL error"));
  }
}

constexpr int kNcclDouble = 8, kNcclSum = 0;  // ncclFloat64, ncclSum (nccl.h)

}  // namespace
}  // namespace sgpx

struct sgpx_multi {
  sgpx_engine_config cfg{};
  std::vector<int> dev;                 // device of shard i
  std::vector<int64_t> b, n;            // rows of shard i
  std::vector<sgpx_ctx*> ctx;
  std::vector<sgpx_engine*> eng;
  std::vector<int> group;               // index into `leaders` of shard i's device
  std::vector<int> leaders;             // first shard of each distinct device
  std::vector<void*> comms;             // one per distinct device (ncclCommInitAll)
  std::vector<cudaEvent_t> ev;          // per shard: its pass is done / the reduced buffer is back
  bool with_grads = false;
  ~sgpx_multi() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    for (auto* e : eng)
      if (e) sgpx_engine_destroy(e);
    for (auto* c : ctx)
      if (c) sgpx_ctx_destroy(c);
    if (!comms.empty() && sgpx::nccl_api().destroy)
      for (void* c : comms)
        if (c) sgpx::nccl_api().destroy(c);
  }
};

namespace sgpx {
namespace {

// Sum the shards' packed buffers (`buf(i)`, `count` doubles) into every shard's buffer.
template <class Buf>
void multi_exchange(sgpx_multi* mu, Buf buf, int64_t count) {
  const int k = int(mu->eng.size());
  for (int i = 0; i < k; ++i) {
    CUDA_OK(cudaSetDevice(mu->dev[i]));
    CUDA_OK(cudaEventRecord(mu->ev[i], mu->ctx[i]->stream));
  }
  // fold same-device shards into their leader (ascending shard order)
  for (int i = 0; i < k; ++i) {
    const int l = mu->leaders[mu->group[i]];
    if (l == i) continue;
    CUDA_OK(cudaSetDevice(mu->dev[l]));
    CUDA_OK(cudaStreamWaitEvent(mu->ctx[l]->stream, mu->ev[i], 0));
    add_into_kernel<<<int(std::min<int64_t>((count + 255) / 256, 1024)), 256, 0, mu->ctx[l]->stream>>>(buf(l), buf(i),
                                                                                                          count);
    CUDA_OK(cudaGetLastError());
  }
  // across devices
  if (mu->leaders.size() > 1) {
    const NcclApi& a = nccl_api();
    nccl_ok(a.group_start(), "ncclGroupStart");
    for (size_t g = 0; g < mu->leaders.size(); ++g) {
      const int l = mu->leaders[g];
      CUDA_OK(cudaSetDevice(mu->dev[l]));
      nccl_ok(a.allreduce(buf(l), buf(l), size_t(count), kNcclDouble, kNcclSum, mu->comms[g], mu->ctx[l]->stream),
              "ncclAllReduce");
    }
    nccl_ok(a.group_end(), "ncclGroupEnd");
  }
  // back to the other shards of each device
  for (int i = 0; i < k; ++i) {
    const int l = mu->leaders[mu->group[i]];
    if (l == i) continue;
    CUDA_OK(cudaSetDevice(mu->dev[l]));
    CUDA_OK(cudaMemcpyAsync(buf(i), buf(l), sizeof(double) * count, cudaMemcpyDeviceToDevice, mu->ctx[l]->stream));
    CUDA_OK(cudaEventRecord(mu->ev[l], mu->ctx[l]->stream));
    CUDA_OK(cudaSetDevice(mu->dev[i]));
    CUDA_OK(cudaStreamWaitEvent(mu->ctx[i]->stream, mu->ev[l], 0));
  }
}

}  // namespace
}  // namespace sgpx

extern "C" {

int sgpx_multi_create(int workers, const int* devices, const sgpx_engine_config* cfg, sgpx_multi** out) {
  return guard([&] {
    require(cfg && out && devices, "multi_create: null argument");
    require(workers >= 1, "Engine: need at least one worker");
    require(cfg->n_global >= workers, "make_partition: more workers than datapoints");
    auto mu = std::make_unique<sgpx_multi>();
    mu->cfg = *cfg;
    const int64_t nn = cfg->n_global, base = nn / workers, rem = nn % workers;  // make_partition (parallel.hpp:28-41)
    int64_t at = 0;
    for (int i = 0; i < workers; ++i) {
      const int64_t len = base + (i < rem ? 1 : 0);
      mu->b.push_back(at);
      mu->n.push_back(len);
      at += len;
      mu->dev.push_back(devices[i]);
    }
    for (int i = 0; i < workers; ++i) {
      int g = -1;
      for (size_t j = 0; j < mu->leaders.size(); ++j)
        if (mu->dev[mu->leaders[j]] == mu->dev[i]) g = int(j);
      if (g < 0) {
        g = int(mu->leaders.size());
        mu->leaders.push_back(i);
      }
      mu->group.push_back(g);
    }
    for (int i = 0; i < workers; ++i) {
      sgpx_ctx* c = nullptr;
      if (sgpx_ctx_create(mu->dev[i], &c) != SGPX_OK) throw CudaError(g_last_error);
      mu->ctx.push_back(c);
      sgpx_engine_config sc = *cfg;
      sc.row_begin = mu->b[i];
      sc.n_local = mu->n[i];
      sgpx_engine* e = nullptr;
      const int rc = sgpx_engine_create(c, &sc, &e);
      if (rc == SGPX_INVALID_ARGUMENT) throw InvalidArgument(g_last_error);
      if (rc != SGPX_OK) throw CudaError(g_last_error);
      if (!getenv("SGPX_DEVICE_COORD")) e->dev_coord = true;  // coordinators run concurrently on their devices
      mu->eng.push_back(e);
      cudaEvent_t ev;
      CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      mu->ev.push_back(ev);
    }
    if (mu->leaders.size() > 1) {
      const NcclApi& a = nccl_api();
      if (!a.init_all || !a.allreduce || !a.group_start || !a.group_end)
        throw NcclError("NCCL (libnccl.so.2) is not available for the multi-GPU exchange");
      std::vector<int> devs;
      for (int l : mu->leaders) devs.push_back(mu->dev[l]);
      mu->comms.assign(devs.size(), nullptr);
      nccl_ok(a.init_all(mu->comms.data(), int(devs.size()), devs.data()), "ncclCommInitAll");
    }
    *out = mu.release();
  });
}

int sgpx_multi_destroy(sgpx_multi* mu) {
  return guard([&] { delete mu; });
}

int sgpx_multi_workers(const sgpx_multi* mu) { return mu ? int(mu->eng.size()) : 0; }

int sgpx_multi_set_data(sgpx_multi* mu, sgpx_cmat x_or_mu, sgpx_cmat s, sgpx_cmat y) {
  return guard([&] {
    require(mu != nullptr, "engine is null");
    auto slice = [](sgpx_cmat a, int64_t r0, int64_t nr) {
      sgpx_cmat v = a;
      v.ld = a.ld ? a.ld : a.rows;
      v.data = a.data ? a.data + r0 : nullptr;
      v.rows = nr;
      return v;
    };
    require(x_or_mu.rows == mu->cfg.n_global && y.rows == mu->cfg.n_global, "Engine: X/Y must hold N rows");
    for (size_t i = 0; i < mu->eng.size(); ++i) {
      const int rc = sgpx_engine_set_data(mu->eng[i], slice(x_or_mu, mu->b[i], mu->n[i]),
                                          mu->cfg.kind == 1 ? slice(s, mu->b[i], mu->n[i]) : s,
                                          slice(y, mu->b[i], mu->n[i]), 0);
      if (rc == SGPX_INVALID_ARGUMENT) throw InvalidArgument(g_last_error);
      if (rc != SGPX_OK) throw CudaError(g_last_error);
    }
  });
}

int sgpx_multi_broadcast(sgpx_multi* mu, const sgpx_kernel_spec* kernel, double beta, sgpx_cmat z, sgpx_cmat m_,
                         sgpx_cmat s) {
  return guard([&] {
    require(mu != nullptr, "engine is null");
    for (size_t i = 0; i < mu->eng.size(); ++i) {
      sgpx_cmat mi{}, si{};
      if (m_.data) {
        require(m_.rows == mu->cfg.n_global && s.rows == mu->cfg.n_global, "broadcast: mu / s must hold N rows");
        mi = m_;
        mi.ld = m_.ld ? m_.ld : m_.rows;
        mi.data = m_.data + mu->b[i];
        mi.rows = mu->n[i];
        si = s;
        si.ld = s.ld ? s.ld : s.rows;
        si.data = s.data + mu->b[i];
        si.rows = mu->n[i];
      }
      const int rc = sgpx_engine_broadcast(mu->eng[i], kernel, beta, z, mi, si, 0);
      if (rc == SGPX_INVALID_ARGUMENT) throw InvalidArgument(g_last_error);
      if (rc == SGPX_NUMERIC) throw NumericError(g_last_error);
      if (rc != SGPX_OK) throw CudaError(g_last_error);
    }
  });
}

int sgpx_multi_evaluate(sgpx_multi* mu, int with_grads, sgpx_eval_result* out, sgpx_mmat d_mu, sgpx_mmat d_s) {
  return guard([&] {
    require(mu != nullptr && out != nullptr, "engine/result is null");
    const auto t0 = std::chrono::steady_clock::now();
    const int k = int(mu->eng.size());
    const int64_t m = mu->cfg.m, q = mu->cfg.q, d = mu->cfg.d;
    for (int i = 0; i < k; ++i) {
      CUDA_OK(cudaSetDevice(mu->dev[i]));
      engine_stats_pass(mu->eng[i]);
    }
    multi_exchange(mu, [&](int i) { return mu->eng[i]->pstats.get<double>(); }, sgpx_packed_stats_count(m, d));
    for (int i = 0; i < k; ++i) {
      CUDA_OK(cudaSetDevice(mu->dev[i]));
      engine_coordinate(mu->eng[i], with_grads != 0);
    }
    if (with_grads) {
      for (int i = 0; i < k; ++i) {
        CUDA_OK(cudaSetDevice(mu->dev[i]));
        engine_grad_pass(mu->eng[i]);
      }
      multi_exchange(mu, [&](int i) { return mu->eng[i]->pgrads.get<double>(); }, sgpx_packed_grads_count(m, q));
    }
    // every shard assembles the same globals; shard 0's are returned, the others checked for errors
    std::vector<double> scratch(size_t(m * (m + d + q) + q + 8));
    for (int i = k - 1; i >= 0; --i) {
      CUDA_OK(cudaSetDevice(mu->dev[i]));
      sgpx_eval_result r = *out;
      if (i != 0) {
        r.psi_y = r.phi_big = r.d_z = r.d_lengthscales = nullptr;
      }
      engine_finish(mu->eng[i], i == 0 ? out : &r);
      if (with_grads && mu->cfg.kind == 1 && d_mu.data && d_s.data) {
        sgpx_mmat a = d_mu, b = d_s;
        a.ld = d_mu.ld ? d_mu.ld : d_mu.rows;
        b.ld = d_s.ld ? d_s.ld : d_s.rows;
        a.data += mu->b[i];
        b.data += mu->b[i];
        a.rows = b.rows = mu->n[i];
        const int rc = sgpx_engine_copy_local_grads(mu->eng[i], a, b);
        if (rc != SGPX_OK) throw CudaError(g_last_error);
      }
    }
    out->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

}  // extern "C"
