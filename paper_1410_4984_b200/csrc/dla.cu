// dla.cu -- fp64 dense linear algebra on the device for the M-sized coordinator and prediction.
//
// Reference: factor_gram / kern_gram / kern_grads (kernels.hpp:83-197), factor_spd / bound_core /
// adjoints_from_core (bound.hpp:52-226), the coordinator block of Engine::evaluate
// (parallel.hpp:378-421) and predict_from_cache (model.hpp:197-217).  The same algebra as
// coordinator.cpp (host), moved onto the stream so an evaluation needs no host round trip between
// its passes and can be captured as one CUDA graph:
//   dla_gemm        C = alpha op(A) op(B) + beta C, 64 x 64 tiles, fixed k order (deterministic)
//   chol_kernel     one CTA: Cholesky with the reference's diagonal escalation schedules
//                   (factor_gram: jitter = f var, f = f0, 10 f0, ... <= 1e-2; factor_spd: + f max|a_ii|,
//                   f = 1e-10 ... 1e-2), log-determinant, status flag.  Right-looking by panels of
//                   32 (16) columns: the panel (rows p0..m) is factored in shared memory, then the
//                   trailing lower triangle is updated once per panel, a warp per 32 x 32 block (the
//                   unblocked column loop is kept for M too large for a shared-memory panel)
//   trinv_kernel    W = L^-1 (lower), one warp per column, the column held in registers (lane i owns
//                   rows i, i + 32, ...), L read column by column (coalesced); a thread per column
//                   above M = 1024
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>

#include "dla.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;

namespace dla {
namespace {

constexpr int kT = 64, kK = 16;

__global__ void __launch_bounds__(256) gemm_kernel(int ta, int tb, int m, int n, int k, double alpha,
                                                   const double* __restrict__ A, int64_t lda,
                                                   const double* __restrict__ B, int64_t ldb, double beta,
                                                   double* __restrict__ C, int64_t ldc) {
  __shared__ double As[kK][kT + 1], Bs[kK][kT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  const int i0 = blockIdx.x * kT, j0 = blockIdx.y * kT;
  double acc[4][4] = {};
  for (int p0 = 0; p0 < k; p0 += kK) {
    for (int e = threadIdx.x; e < kK * kT; e += 256) {
      const int pp = e / kT, ii = e % kT;
      const int i = i0 + ii, p = p0 + pp;
      double a = 0.0;
      if (i < m && p < k) a = ta ? A[p + int64_t(i) * lda] : A[i + int64_t(p) * lda];
      As[pp][ii] = a;
      const int j = j0 + ii;
      double b = 0.0;
      if (j < n && p < k) b = tb ? B[j + int64_t(p) * ldb] : B[p + int64_t(j) * ldb];
      Bs[pp][ii] = b;
    }
    __syncthreads();
#pragma unroll
    for (int pp = 0; pp < kK; ++pp) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[pp][tx + 16 * u];
        b[u] = Bs[pp][ty + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = i0 + tx + 16 * u, j = j0 + ty + 16 * v;
      if (i < m && j < n) {
        double* c = C + i + int64_t(j) * ldc;
        *c = alpha * acc[u][v] + (beta == 0.0 ? 0.0 : beta * *c);
      }
    }
}

// In-place lower Cholesky of the m x m working copy `w` (lower triangle used, upper zeroed),
// right-looking by columns; all threads of the CTA.  Returns false on a non-positive / NaN pivot.
__device__ bool chol_inplace(double* w, int m, int64_t ld, double* s_piv) {
  for (int j = 0; j < m; ++j) {
    if (threadIdx.x == 0) {
      const double d = w[j + int64_t(j) * ld];
      s_piv[0] = (d > 0.0) ? sqrt(d) : -1.0;
    }
    __syncthreads();
    const double ljj = s_piv[0];
    if (!(ljj > 0.0)) return false;
    const double inv = 1.0 / ljj;
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) w[i + int64_t(j) * ld] *= inv;
    __syncthreads();
    if (threadIdx.x == 0) w[j + int64_t(j) * ld] = ljj;
    // trailing update of the lower triangle: w[i][c] -= l_ij l_cj, j < c <= i
    const int rem = m - j - 1;
    for (int64_t e = threadIdx.x; e < int64_t(rem) * rem; e += blockDim.x) {
      const int r = int(e / rem), c = int(e % rem);
      if (c > r) continue;
      const int i = j + 1 + r, col = j + 1 + c;
      w[i + int64_t(col) * ld] -= w[i + int64_t(j) * ld] * w[col + int64_t(j) * ld];
    }
    __syncthreads();
  }
  return true;
}

// Blocked form of chol_inplace: panels of nbm (32, or 16 for large M) columns.  panel: shared
// column-major (m - p0) x nbm with column stride RS >= m (thread-per-row accesses are conflict-free,
// column reads by a warp broadcast).  Same result up to the order of the trailing-update sums.
__device__ bool chol_blocked(double* w, int m, int64_t ld, double* panel, double* s_piv, int nbm, int RS) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int p0 = 0; p0 < m; p0 += nbm) {
    const int nb = min(nbm, m - p0), rows = m - p0;
    for (int c = warp; c < nbm; c += nwarps)
      for (int r = lane; r < rows; r += 32) panel[c * RS + r] = c < nb ? w[p0 + r + int64_t(p0 + c) * ld] : 0.0;
    __syncthreads();
    // panel factor, thread per panel row: the rows' entries right of column j are updated from the
    // still-unscaled column j (times 1 / l_jj), then column j is scaled after a barrier
    for (int j = 0; j < nb; ++j) {
      if (threadIdx.x == 0) {
        const double d = panel[j * RS + j];
        s_piv[0] = (d > 0.0) ? sqrt(d) : -1.0;
      }
      __syncthreads();
      const double ljj = s_piv[0];
      if (!(ljj > 0.0)) return false;
      const double inv = 1.0 / ljj;
      for (int r = j + 1 + threadIdx.x; r < rows; r += blockDim.x) {
        const double lrj = panel[j * RS + r] * inv;
        const int cmax = min(nb - 1, r);
#pragma unroll 4
        for (int c = j + 1; c <= cmax; ++c) panel[c * RS + r] -= lrj * (panel[j * RS + c] * inv);
      }
      __syncthreads();
      for (int r = j + threadIdx.x; r < rows; r += blockDim.x)
        panel[j * RS + r] = r == j ? ljj : panel[j * RS + r] * inv;
    }
    __syncthreads();
    for (int c = warp; c < nb; c += nwarps)
      for (int r = lane; r < rows; r += 32) w[p0 + r + int64_t(p0 + c) * ld] = r < c ? 0.0 : panel[c * RS + r];
    // trailing lower triangle: w[i][c] -= sum_k P[i][k] P[c][k] for p0 + nb <= c <= i < m.  A warp per
    // 32 x 32 block (I >= J), each lane a 4 x 8 register tile (lane & 7 -> rows, lane >> 3 -> columns):
    // 12 shared loads per 32 FMAs, k ascending
    const int t0 = nb, tr = rows - nb;
    const int nbk = (tr + 31) / 32, nblk = nbk * (nbk + 1) / 2;
    const int lr = lane & 7, lc = lane >> 3;
    for (int b = warp; b < nblk; b += nwarps) {
      int I = int((sqrt(8.0 * double(b) + 1.0) - 1.0) * 0.5);
      while (I * (I + 1) / 2 > b) --I;
      while ((I + 1) * (I + 2) / 2 <= b) ++I;
      const int J = b - I * (I + 1) / 2;
      const int i0 = I * 32 + lr * 4, j0 = J * 32 + lc * 8;  // trailing-relative
      double acc[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = 0.0;
      for (int k = 0; k < nb; ++k) {
        const double* col = panel + k * RS + t0;
        double av[4], bv[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) av[u] = i0 + u < tr ? col[i0 + u] : 0.0;
#pragma unroll
        for (int v = 0; v < 8; ++v) bv[v] = j0 + v < tr ? col[j0 + v] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 8; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
      }
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int jl = j0 + v;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int il = i0 + u;
          if (jl < tr && il < tr && il >= jl) w[p0 + t0 + il + int64_t(p0 + t0 + jl) * ld] -= acc[u][v];
        }
      }
    }
    __syncthreads();
  }
  return true;
}

// mode 0 (factor_gram, kernels.hpp:177-197): diag += f * var, f = f0, then x10 (0 -> 1e-6) while
// f < 1e-2, failure after 1e-2.  mode 1 (factor_spd, bound.hpp:52-62): first the plain matrix, then
// diag += f * max_i |a_ii| for f = 1e-10, 1e-9, ..., 1e-2.
// a: m x m input (lower and upper valid), out: L (upper zeroed); info[0] = status (0 ok, 1 failed),
// out_scal[0] = log det, out_scal[1] = jitter factor used (mode 0) / shift used (mode 1).
__global__ void __launch_bounds__(512) chol_kernel(const double* __restrict__ a, int m, double* __restrict__ L,
                                                    int mode, double f0, double var, double* __restrict__ out_scal,
                                                    int* __restrict__ info, int nbm) {
  extern __shared__ double panel[];
  __shared__ double s_piv[1], s_red[512];
  const int64_t ld = m;
  double scale = 0.0;
  if (mode == 1) {
    double mx = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) mx = fmax(mx, fabs(a[i + int64_t(i) * ld]));
    s_red[threadIdx.x] = mx;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) s_red[threadIdx.x] = fmax(s_red[threadIdx.x], s_red[threadIdx.x + w]);
      __syncthreads();
    }
    scale = s_red[0];
    __syncthreads();
  }
  double f = mode == 0 ? f0 : 0.0;
  bool ok = false;
  for (int attempt = 0; attempt < 32; ++attempt) {
    const double shift = mode == 0 ? f * var : f * scale;
    for (int j = threadIdx.x >> 5; j < m; j += blockDim.x >> 5)
      for (int i = threadIdx.x & 31; i < m; i += 32) {
        const int64_t e = i + int64_t(j) * m;
        L[e] = i < j ? 0.0 : a[e] + (i == j ? shift : 0.0);
      }
    __syncthreads();
    ok = nbm ? chol_blocked(L, m, ld, panel, s_piv, nbm, m | 1) : chol_inplace(L, m, ld, s_piv);
    __syncthreads();
    if (ok) break;
    if (mode == 0) {
      if (f >= 1e-2) break;
      f = f == 0.0 ? 1e-6 : f * 10.0;
    } else {
      f = f == 0.0 ? 1e-10 : f * 10.0;  // for (f = 1e-10; f <= 1e-2; f *= 10) (bound.hpp:57)
      if (!(f <= 1e-2)) break;
    }
  }
  if (threadIdx.x == 0) {
    info[0] = ok ? 0 : 1;
    out_scal[1] = f;
  }
  // log det = 2 sum log L_ii (fixed tree)
  double s = 0.0;
  if (ok)
    for (int i = threadIdx.x; i < m; i += blockDim.x) s += log(L[i + int64_t(i) * ld]);
  s_red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s_red[threadIdx.x] += s_red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out_scal[0] = 2.0 * s_red[0];
}

// W = L^-1 (lower triangular): thread j solves L w = e_j by column-oriented forward substitution
// (the order of coordinator.cpp's chol_inverse).
__global__ void trinv_kernel(const double* __restrict__ L, int m, double* __restrict__ W) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double* x = W + int64_t(j) * m;
  for (int i = 0; i < m; ++i) x[i] = i == j ? 1.0 : 0.0;
  for (int k = j; k < m; ++k) {
    const double xk = x[k] / L[k + int64_t(k) * m];
    x[k] = xk;
    const double* lk = L + int64_t(k) * m;
    for (int i = k + 1; i < m; ++i) x[i] -= lk[i] * xk;
  }
}

// Same substitution, warp per column j: lane l owns x[l + 32 t], t < T (T * 32 >= m).  Step k
// broadcasts x_k / L_kk from its owner and updates the rows below with column k of L.
template <int T>
__global__ void __launch_bounds__(64) trinv_warp_kernel(const double* __restrict__ L, int m, double* __restrict__ W) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * 2 + (threadIdx.x >> 5);
  if (j >= m) return;
  double x[T];
#pragma unroll
  for (int t = 0; t < T; ++t) x[t] = (lane + 32 * t == j) ? 1.0 : 0.0;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    if (32 * t + 31 < j || 32 * t >= m) continue;
    const int kd = 32 * t + lane;
    const double rd = kd < m ? 1.0 / L[kd + int64_t(kd) * m] : 0.0;  // 1 / L_kk of the slot's rows
#pragma unroll 4
    for (int l = 0; l < 32; ++l) {
      const int k = 32 * t + l;
      if (k < j || k >= m) continue;
      const double xk = __shfl_sync(0xffffffffu, x[t], l) * __shfl_sync(0xffffffffu, rd, l);
      if (lane == l) x[t] = xk;
      const double* lk = L + int64_t(k) * m;
#pragma unroll
      for (int u = t; u < T; ++u) {
        const int i = lane + 32 * u;
        if (i > k && i < m) x[u] = fma(-lk[i], xk, x[u]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int i = lane + 32 * t;
    if (i < m) W[i + int64_t(j) * m] = x[t];
  }
}

}  // namespace

int gemm(bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int64_t lda, const double* B,
         int64_t ldb, double beta, double* C, int64_t ldc, cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  dim3 grid(unsigned((m + kT - 1) / kT), unsigned((n + kT - 1) / kT));
  gemm_kernel<<<grid, 256, 0, st>>>(ta ? 1 : 0, tb ? 1 : 0, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int cholesky(const double* a, int m, double* L, int mode, double f0, double var, double* out_scal, int* info,
             cudaStream_t st) {
  // panel width 32 while the (m x 34) panel fits the opt-in shared memory, else 16, else unblocked
  constexpr size_t kSmemMax = 200 * 1024;
  int nbm = 0;
  if (sizeof(double) * size_t(m | 1) * 32 <= kSmemMax) nbm = 32;
  else if (sizeof(double) * size_t(m | 1) * 16 <= kSmemMax) nbm = 16;
  const size_t smem = nbm ? sizeof(double) * size_t(m | 1) * nbm : 0;
  if (nbm) {
    static std::atomic<uint64_t> attr_set{0};  // per-device one-time opt-in (the largest size asked for)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 3;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (!(attr_set.load() & bit)) {
      if (cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemMax)) != cudaSuccess)
        return 3;
      attr_set.fetch_or(bit);
    }
  }
  chol_kernel<<<1, 512, smem, st>>>(a, m, L, mode, f0, var, out_scal, info, nbm);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int trinv(const double* L, int m, double* W, cudaStream_t st) {
  const unsigned g = unsigned((m + 1) / 2);
  if (m <= 128) trinv_warp_kernel<4><<<g, 64, 0, st>>>(L, m, W);
  else if (m <= 256) trinv_warp_kernel<8><<<g, 64, 0, st>>>(L, m, W);
  else if (m <= 512) trinv_warp_kernel<16><<<g, 64, 0, st>>>(L, m, W);
  else if (m <= 1024) trinv_warp_kernel<32><<<g, 64, 0, st>>>(L, m, W);
  else trinv_kernel<<<(m + 127) / 128, 128, 0, st>>>(L, m, W);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace dla
}  // namespace sgpx
