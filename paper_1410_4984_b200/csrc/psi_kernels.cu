// psi_kernels.cu -- dispatch of the psi-statistics passes and the small shared kernels.
//
// Reference hot path: proj/include/sgp/psi_stats.hpp:108-326 (detail::sweep_stats), plus the KL
// partial / KL gradients of Worker::pass (parallel.hpp:148-149, 163-166).  One evaluation runs in
// one of three modes (psi_kernels.cuh), chosen on the host from the inducing points:
//   fast / precise  psi1 tiles (psi1_tile.cu, psi1_kernels.cu) + row-tile tcgen05 psi2
//                   (psi_rowtile.cu), two or three fp16 pieces per exponent feature
//   direct          direct-difference kernels with fp64 exponents (psi_direct.cu)
// Every cross-CTA sum is fp64 and runs in a fixed order in a second small kernel, so results are
// bitwise reproducible run to run.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "psi_common.cuh"
#include "psi_kernels.cuh"

namespace sgpx {
namespace {

std::atomic<int64_t> g_launches{0};
using namespace dev;

// Fixed-order column sums of nparts partial rows: a block covers 32 columns with 8 warps, warp w
// summing rows w, w + 8, ... (coalesced across the columns), then the 8 partial sums in order.
// Launch with 256 threads and ceil(count / 32) blocks.
__device__ __forceinline__ bool colsum8(const double* __restrict__ part, int64_t pstride, int nparts, int64_t count,
                                        int64_t& k, double& sum) {
  __shared__ double red[8][32];
  const int kk = threadIdx.x & 31, w = threadIdx.x >> 5;
  k = int64_t(blockIdx.x) * 32 + kk;
  double s = 0.0;
  if (k < count)
    for (int c = w; c < nparts; c += 8) s += part[c * pstride + k];
  red[w][kk] = s;
  __syncthreads();
  if (w != 0 || k >= count) return false;
  sum = red[0][kk];
  for (int i = 1; i < 8; ++i) sum += red[i][kk];
  return true;
}

// Fixed-order reduction of the per-CTA forward partials into the packed stats vector.
__global__ void __launch_bounds__(256) fwd_reduce_kernel(const double* __restrict__ part, int64_t pstride, int nparts,
                                                         int64_t count, double* __restrict__ packed, double phi_val,
                                                         double n_count) {
  int64_t k;
  double s;
  if (colsum8(part, pstride, nparts, count, k, s)) {
    if (k == 0)
      packed[1] = s;
    else if (k == 1)
      packed[3] = s;
    else
      packed[k + 2] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    packed[0] = phi_val;
    packed[2] = n_count;
  }
}

__global__ void psi1_matrix_kernel(PsiConst P, double* __restrict__ out, int64_t ld_out) {
  const int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int mm = blockIdx.y;
  if (n >= P.n || mm >= P.m) return;
  double e = 0.0, lc = 0.0;
  for (int q = 0; q < P.q; ++q) {
    const double mu = P.mu[q * P.ld_mu + n], s = P.s[q * P.ld_s + n];
    const double l2 = P.ls[q] * P.ls[q];
    const double df = mu - P.z64[mm + int64_t(q) * P.m];
    e += df * df / (s + l2);
    lc += log1p(s / l2);
  }
  out[mm * ld_out + n] = P.variance_d * exp(-0.5 * lc - 0.5 * e);
}

// Two-level fixed-order reduction of `rows` partial rows: row groups in parallel (level 1), then
// the group sums in ascending order (level 2).  tmp: kReduceGroups * pstride doubles.
constexpr int kReduceGroups = 64;
__global__ void rows_partial_kernel(const double* __restrict__ part, int64_t pstride, int rows, int groups,
                                    double* __restrict__ tmp) {
  const int g = blockIdx.y;
  const int r0 = int(int64_t(g) * rows / groups), r1 = int(int64_t(g + 1) * rows / groups);
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < pstride; k += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int r = r0; r < r1; ++r) s += part[int64_t(r) * pstride + k];
    tmp[int64_t(g) * pstride + k] = s;
  }
}
__global__ void rows_final_bwd_kernel(const double* __restrict__ tmp, int groups, int64_t pstride,
                                      double* __restrict__ packed, double dvar0) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < pstride; k += int64_t(gridDim.x) * blockDim.x) {
    double s = k == 0 ? dvar0 : 0.0;
    for (int g = 0; g < groups; ++g) s += tmp[int64_t(g) * pstride + k];
    packed[k] = s;
  }
}

// ---------------------------------------------------------------------------
// Host-side dispatch over the instantiated latent dimensions.
// ---------------------------------------------------------------------------
constexpr int kQs[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32};

int pick_q(int q) {
  for (int v : kQs)
    if (v >= q) return v;
  return -1;
}

// Envelope of the row-tile path in Tz = max_a sum_q ((z_a - c) / l)^2 (tools/envelope.py,
// profiles/accuracy/r02_envelope_modes.log), for the tolerances the parity tests assert (norm-wise
// 1e-5 statistics / 5e-5 gradients, element-wise rel_err <= 1e-4): latent (expected) mode, two pieces
// up to Tz = 150 (worst measured: 1.6e-5 norm d Z at 133), three pieces up to 600 (6.6e-5 element d l
// at 221, bimodal Z); deterministic (SGPR) mode, whose narrower kernel cancels harder, three pieces
// up to Tz = 60 (1.2e-4 element d l already at 133).  Beyond, the direct kernels run.
constexpr double kTzFast = 150.0;
constexpr double kTzPrecise = 600.0;
constexpr double kTzPreciseDet = 60.0;

int env_mode() {
  static const int v = [] {
    const char* e = getenv("SGPX_PSI_MODE");
    if (!e) return kModeAuto;
    if (!strcmp(e, "fast")) return kModeFast;
    if (!strcmp(e, "precise")) return kModePrecise;
    if (!strcmp(e, "direct")) return kModeDirect;
    if (!strcmp(e, "syrk")) return kModeSyrk;
    return kModeAuto;
  }();
  return v;
}

}  // namespace

std::atomic<int64_t> g_tc_launches{0};
int64_t launches_issued() { return g_launches.load() + g_tc_launches.load(); }
void launches_add(int64_t n) { g_tc_launches.fetch_add(n); }
int instantiated_q(int q) { return pick_q(q); }

int64_t bwd_reduce_tmp_doubles(int64_t pstride) { return int64_t(kReduceGroups) * pstride; }

int bwd_reduce_rows(const double* part, int64_t pstride, int rows, double* packed, double dvar0, double* tmp,
                    void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int groups = std::max(1, std::min(kReduceGroups, rows));
  const int cb = int(std::min<int64_t>((pstride + 255) / 256, 64));
  rows_partial_kernel<<<dim3(cb, groups), 256, 0, st>>>(part, pstride, rows, groups, tmp);
  rows_final_bwd_kernel<<<cb, 256, 0, st>>>(tmp, groups, pstride, packed, dvar0);
  g_launches.fetch_add(2);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Row-tile tensor-core psi2 where it is instantiated.  The deterministic (SGPR) kernel is narrower
// (den = 1/l^2, no 2S), so the assembly from the exponent-as-GEMM sums cancels harder: it runs in
// the precise mode and only up to Q = 16 (d_l <= 2.1e-5; 6e-5 .. 9e-5 at Q = 18 / 20,
// profiles/accuracy/r01_q_sweep_*.log).
bool use_rt(const PsiConst& P) { return (P.expected || instantiated_q(P.q) <= 16) && rt_supported(P); }

double psi_z_spread(const PsiConst& P, const double* z, int64_t m) {
  double tz = 0.0;
  for (int64_t a = 0; a < m; ++a) {
    double s = 0.0;
    for (int q = 0; q < P.q; ++q) {
      const double v = (z[a + q * m] - P.center[q]) / P.ls[q];
      s += v * v;
    }
    tz = std::max(tz, s);
  }
  return tz;
}

int psi_select_mode(const PsiConst& P, const double* z, int64_t m, int requested) {
  if (P.q > kMaxQ) return -1;
  int req = requested != kModeAuto ? requested : env_mode();
  // deterministic inputs: the Knm-tile SYRK unless another mode is asked for (accurate at any spread)
  if (!P.expected && (req == kModeAuto || req == kModeSyrk) && syrk_supported(P)) return kModeSyrk;
  if (req == kModeSyrk) req = kModeAuto;  // latent inputs have no SYRK form
  if (!use_rt(P)) return kModeDirect;
  if (req == kModeDirect) return kModeDirect;
  const double tz = psi_z_spread(P, z, m);
  if (req == kModeFast || req == kModePrecise) return tz <= 5.0e4 ? req : kModeDirect;  // features within the fp16 range
  if (!P.expected) return tz <= kTzPreciseDet ? kModePrecise : kModeDirect;  // SGPR: precise mode only
  if (tz <= kTzFast) return kModeFast;
  if (tz <= kTzPrecise) return kModePrecise;
  return kModeDirect;
}

static bool is_syrk(const PsiConst& P) { return P.mode == kModeSyrk; }
static bool is_direct(const PsiConst& P) { return !is_syrk(P) && (P.mode == kModeDirect || !use_rt(P)); }

const double* fwd_region(const PsiConst& P, const double* fwd_part, int num_sms) {
  if (is_direct(P) || is_syrk(P)) return fwd_part;
  return fwd_part + int64_t(psi1_fwd_rows(P, num_sms)) * fwd_part_count(P.m, P.d);
}

double* fwd_pair_sums(const PsiConst& P, double* region, int num_sms, int64_t* count) {
  if (is_syrk(P)) {  // the SYRK backward needs no forward sums
    *count = 0;
    return region;
  }
  if (is_direct(P)) return direct_fwd_pair_sums(P, region, num_sms, count);
  return rt_fwd_pair_sums(P, region, num_sms, count);
}

double* bwd_rt_region(const PsiConst& P, double* part, int num_sms) {
  const int rows = (P.n > 0 ? psi1_bwd_rows(P, num_sms) : 0) + 1;  // as psi_backward lays it out
  return part + int64_t(rows) * bwd_part_count(P.m, P.q);
}

const float* fwd_pair_operand(const PsiConst& P, const double* region, int num_sms) {
  if (is_syrk(P) || is_direct(P)) return nullptr;
  return rt_fwd_pair_operand(P, region, num_sms);
}

int psi_forward(const PsiConst& P, double* part, double* packed, int* err_flag, int num_sms, void* stream,
                LaunchGeom* geom, void* ev_begin, void* ev_end) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LaunchGeom g{};
  if (int rc = plan_forward(P, num_sms, &g)) return rc;
  if (is_syrk(P)) {
    if (ev_begin) record_event(ev_begin, st);
    if (int rc = syrk_forward(P, part, packed, err_flag, num_sms, stream)) return rc;
    if (ev_end) record_event(ev_end, st);
    if (geom) *geom = g;
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  if (is_direct(P)) {
    if (!direct_supported(P)) return 1;
    if (ev_begin) record_event(ev_begin, st);
    if (int rc = direct_forward(P, part, packed, err_flag, P.expected, num_sms, stream)) return rc;
    if (ev_end) record_event(ev_end, st);
    if (geom) *geom = g;
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  const int64_t pstride = fwd_part_count(P.m, P.d);
  const int g1 = psi1_fwd_rows(P, num_sms);
  if (g1 > 0 && cudaMemsetAsync(part, 0, sizeof(double) * pstride * g1, st) != cudaSuccess) return 3;
  if (ev_begin) record_event(ev_begin, st);
  if (g1 > 0) {
    if (int rc = psi1_forward(P, part, pstride, g1, err_flag, stream, 1)) return rc;
  }
  fwd_reduce_kernel<<<int((pstride + 31) / 32), 256, 0, st>>>(part, pstride, g1, pstride, packed,
                                                                 double(P.n) * P.variance_d, double(P.n));
  g_launches.fetch_add(1);
  if (int rc = rt_forward(P, part + int64_t(g1) * pstride, packed, num_sms, stream)) return rc;
  if (ev_end) record_event(ev_end, st);
  if (geom) *geom = g;
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

bool psi_backward_phased(const PsiConst& P) { return !is_syrk(P) && !is_direct(P); }

int psi_backward(const PsiConst& P, const BwdConst& B, double* part, double* packed, int num_sms, void* stream,
                 LaunchGeom* geom, void* ev_begin, void* ev_end, int phase, void* reduce_stream, void* reduce_event,
                 int psi1_grid_cap) {
  if (!B.fwd_rt) return 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LaunchGeom g{};
  if (int rc = plan_backward(P, num_sms, &g)) return rc;
  if (is_syrk(P)) {
    if (ev_begin) record_event(ev_begin, st);
    if (int rc = syrk_backward(P, B, part, packed, num_sms, stream)) return rc;
    if (ev_end) record_event(ev_end, st);
    if (geom) *geom = g;
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  if (is_direct(P)) {
    if (ev_begin) record_event(ev_begin, st);
    if (int rc = direct_backward(P, B, part, packed, num_sms, stream)) return rc;
    if (ev_end) record_event(ev_end, st);
    if (geom) *geom = g;
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  const int64_t pstride = bwd_part_count(P.m, P.q);
  const int r1 = P.n > 0 ? psi1_bwd_rows(P, num_sms) : 0, rows = r1 + 1;
  if (phase != 2) {
    if (cudaMemsetAsync(part, 0, sizeof(double) * pstride * rows, st) != cudaSuccess) return 3;
    if (ev_begin) record_event(ev_begin, st);
    // psi1 first: it writes d_mu / d_s (psi1 + KL parts); the psi2 kernel accumulates into them
    if (r1 > 0) {
      const int g1 = psi1_grid_cap > 0 ? std::min(r1, psi1_grid_cap) : r1;
      if (int rc = psi1_backward(P, B, part, pstride, g1, stream)) return rc;
    }
    if (phase == 1) return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  if (int rc = rt_backward(P, B, part + int64_t(rows) * pstride, part + int64_t(r1) * pstride, num_sms, stream))
    return rc;
  if (ev_end) record_event(ev_end, st);
  const int64_t rt_rows = (rt_bwd_doubles(P, num_sms) + pstride - 1) / pstride;
  double* tmp = part + (int64_t(rows) + rt_rows) * pstride;
  if (reduce_stream && reduce_event) {  // off the pass's stream: the next sub-shard's kernels do not wait
    cudaStream_t rs = static_cast<cudaStream_t>(reduce_stream);
    if (cudaEventRecord(static_cast<cudaEvent_t>(reduce_event), st) != cudaSuccess ||
        cudaStreamWaitEvent(rs, static_cast<cudaEvent_t>(reduce_event), 0) != cudaSuccess)
      return 3;
    if (int rc = bwd_reduce_rows(part, pstride, rows, packed, B.d_phi * double(P.n), tmp, rs)) return rc;
  } else if (int rc = bwd_reduce_rows(part, pstride, rows, packed, B.d_phi * double(P.n), tmp, stream)) {
    return rc;
  }
  if (geom) *geom = g;
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int plan_forward(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  const int64_t pstride = fwd_part_count(P.m, P.d);
  if (is_syrk(P)) {
    *geom = LaunchGeom{int((syrk_fwd_doubles(P, num_sms) + pstride - 1) / pstride), 256, 0};
    return 0;
  }
  if (is_direct(P)) {
    *geom = LaunchGeom{int((direct_fwd_doubles(P, num_sms) + pstride - 1) / pstride), 128, 0};
    return 0;
  }
  // partial rows: psi1 rows + the row-tile region
  const int64_t extra = (rt_fwd_doubles(P, num_sms) + pstride - 1) / pstride;
  *geom = LaunchGeom{int(psi1_fwd_rows(P, num_sms) + extra), 448, 0};
  return 0;
}

int plan_backward(const PsiConst& P, int num_sms, LaunchGeom* geom) {
  const int64_t pstride = bwd_part_count(P.m, P.q);
  if (is_syrk(P)) {
    *geom = LaunchGeom{int((syrk_bwd_doubles(P, num_sms) + pstride - 1) / pstride), 256, 0};
    return 0;
  }
  if (is_direct(P)) {
    *geom = LaunchGeom{int((direct_bwd_doubles(P, num_sms) + pstride - 1) / pstride), 128, 0};
    return 0;
  }
  // psi1 rows (8 per CTA) + 1 psi2 row + the row-tile scratch
  const int r1 = P.n > 0 ? psi1_bwd_rows(P, num_sms) : 0;
  const int64_t extra = (rt_bwd_doubles(P, num_sms) + pstride - 1) / pstride +
                        (bwd_reduce_tmp_doubles(pstride) + pstride - 1) / pstride;
  *geom = LaunchGeom{int(r1 + 1 + extra), 448, 0};
  return 0;
}

int psi1_matrix(const PsiConst& P, double* out, int64_t ld_out, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (P.n == 0 || P.m == 0) return 0;
  dim3 grid(unsigned((P.n + 127) / 128), unsigned(P.m));
  psi1_matrix_kernel<<<grid, 128, 0, st>>>(P, out, ld_out);
  g_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace sgpx
