// syrk.cu -- deterministic inputs (sparse GP regression) as Knm tiles and tensor-core GEMMs.
//
// Reference: the deterministic branch of sweep_stats (psi_stats.hpp:160-167, 256-273, 305-315), whose
// psi2 term is the product of two kernel values, v_n,ab = var^2 exp(-1/2 sum_q ((x-za)^2 + (x-zb)^2)/l^2)
// = K_na K_nb (kernels.hpp:56-78), so that
//     Phi = K^T K,   Psi = K^T Y,
//     dL/dK = G = 2 K U + Y dPsi^T          (U = dL/dPhi, symmetric)
//     d Z_aq = sum_n H_na (x_nq - z_aq) / l_q^2,  d l_q = sum_na H_na (x_nq - z_aq)^2 / l_q^3,
//     d var = sum_na H_na / var + d_phi N,   H = G o K          (the kern_grads form, kernels.hpp:145-161)
// The reference spends one exp per (n, pair); this path spends one per (n, m) and moves the N M^2
// work onto the tensor cores.
//
// Per chunk of kChunk datapoints:
//   knm_split_kernel   K_na in fp64 (direct differences, fp64 exp), split for split-TF32 GEMMs into
//                      big = tf32(K) and small = K - big (fp32; big + small carries ~2^-35 of K),
//                      with Y appended as extra columns: B = [K | Y]
//   forward            C = K^T B by three cuBLAS TF32 GEMMs (big.big + big.small + small.big), batched
//                      over kSub-row sub-chunks so fp32 accumulates over kSub rows only, the sub-chunk
//                      results added into an fp64 accumulator in order -> Phi (upper triangle) and Psi
//   backward           G^T = [2U ; dPsi^T]^T [K | Y]^T by the same three-pass split (inner dimension
//                      M + D padded to a multiple of 4)
//   syrk_reduce_kernel H = G o K (K = big + small of the same chunk matrix) and the d Z / d l / d var
//                      sums as centred fp64 moments (lane per inducing point, fixed order)
// Precision mode: split-TF32 tensor-core GEMMs with fp32 accumulation inside a sub-chunk, fp64 across
// sub-chunks; exponents, K and every gradient contraction in fp64.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <thread>

#include "psi_common.cuh"
#include "psi_kernels.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;
namespace {

constexpr int64_t kChunk = 65536;  // datapoints per chunk (Knm tile in HBM)
constexpr int64_t kSub = 512;      // fp32 accumulation length of the forward GEMMs (batched sub-chunks)
constexpr int kBatch = int(kChunk / kSub);
constexpr double kL2e = 1.4426950408889634;

// 2^x to ~2e-13 relative (degree-10 Taylor on the rint split, |t| <= ln2 / 2): K only needs the
// ~2^-35 that its big + small split carries.
__device__ __forceinline__ double exp2_k(double x) {
  if (!(x > -1020.0)) return 0.0;
  const double j = rint(x);
  const double t = (x - j) * 0.69314718055994530942;
  double p = 1.0 / 3628800.0;
  p = fma(p, t, 1.0 / 362880.0);
  p = fma(p, t, 1.0 / 40320.0);
  p = fma(p, t, 1.0 / 5040.0);
  p = fma(p, t, 1.0 / 720.0);
  p = fma(p, t, 1.0 / 120.0);
  p = fma(p, t, 1.0 / 24.0);
  p = fma(p, t, 1.0 / 6.0);
  p = fma(p, t, 0.5);
  p = fma(p, t, 1.0);
  p = fma(p, t, 1.0);
  return p * __hiloint2double((int(j) + 1023) << 20, 0);
}

__device__ __forceinline__ void split_tf32(double v, float& big, float& small) {
  const float f = float(v);
  uint32_t u = __float_as_uint(f);
  u = (u + 0x1000u) & 0xFFFFE000u;  // round to the 10-bit tf32 mantissa
  big = __uint_as_float(u);
  small = float(v - double(big));
}

// K_na = var exp(-1/2 sum_q ((x_nq - z_aq) / l_q)^2) for rows [n0, n0 + nc) -> big / small [nc][ldc]
// column-major (ld = nc), columns [0, M) = K, [M, M + D) = Y, [M + D, ncols) zero padding.  Grid:
// (row blocks of 256, column blocks of kCols); the row's x / l in registers, z_a / l broadcast.
constexpr int kCols = 16;
template <int Q>
__global__ void __launch_bounds__(256) knm_split_kernel(PsiConst P, int64_t n0, int64_t nc, int ncols,
                                                        float* __restrict__ big, float* __restrict__ small,
                                                        double2* __restrict__ xp) {
  __shared__ double s_z[kCols][Q];  // z_c / l for the block's columns
  const int m = P.m, c0 = int(blockIdx.y) * kCols;
  for (int i = threadIdx.x; i < kCols * Q; i += blockDim.x) {
    const int cc = i / Q, q = i % Q, c = c0 + cc;
    s_z[cc][q] = (c < m && q < P.q) ? P.z64[c + int64_t(q) * m] / P.ls[q] : 0.0;
  }
  __syncthreads();
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= nc) return;
  const int64_t n = n0 + r;
  const bool valid = n < P.n;
  const double lvar = log2(P.variance_d);
  double xs[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) xs[q] = (valid && q < P.q) ? P.mu[q * P.ld_mu + n] / P.ls[q] : 0.0;
  if (xp && blockIdx.y == 0) {  // (x', x'^2) rows for syrk_reduce_kernel, x' = (x - c) / l
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const double v = (valid && q < P.q) ? (P.mu[q * P.ld_mu + n] - P.center[q]) / P.ls[q] : 0.0;
      xp[r * Q + q] = make_double2(v, v * v);
    }
  }
  const int c1 = min(ncols, c0 + kCols);
  for (int c = c0; c < c1; ++c) {
    double v = 0.0;
    if (valid) {
      if (c < m) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const double d = xs[q] - s_z[c - c0][q];
          s = fma(d, d, s);
        }
        v = exp2_k(lvar - 0.5 * kL2e * s);
      } else if (c < m + P.d) {
        v = P.y[int64_t(c - m) * P.ld_y + n];
      }
    }
    float b, sm;
    split_tf32(v, b, sm);
    big[r + int64_t(c) * nc] = b;
    small[r + int64_t(c) * nc] = sm;
  }
}

// acc (fp64, M x (M + D)) += sum of the nb sub-chunk results (fp32), ascending sub-chunk order
__global__ void acc_add_kernel(double* __restrict__ acc, const float* __restrict__ c, int nb, int64_t count) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    double s = acc[i];
    for (int b = 0; b < nb; ++b) s += double(c[int64_t(b) * count + i]);
    acc[i] = s;
  }
}

// packed[4 + p] = Phi (m1-major upper triangle, symmetrised), packed[4 + P + a + d M] = Psi; yy and phi
__global__ void syrk_pack_kernel(PsiConst P, const double* __restrict__ acc, double* __restrict__ packed) {
  const int m = P.m;
  const int64_t npairs = int64_t(m) * (m + 1) / 2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npairs + int64_t(m) * P.d;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (i < npairs) {
      int a = 0;
      int64_t rem = i;
      while (rem >= m - a) {
        rem -= m - a;
        ++a;
      }
      const int b = a + int(rem);
      packed[4 + i] = 0.5 * (acc[a + int64_t(b) * m] + acc[b + int64_t(a) * m]);
    } else {
      const int64_t k = i - npairs;  // a + d M
      packed[4 + i] = acc[int64_t(m) * m + k];
    }
  }
}

// yy = sum y^2, validation flag (non-finite x / y), per-block partials
__global__ void syrk_rows_kernel(PsiConst P, double* __restrict__ part, int* __restrict__ err) {
  __shared__ double red[256];
  double yy = 0.0;
  int flag = 0;
  for (int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; n < P.n; n += int64_t(gridDim.x) * blockDim.x) {
    for (int q = 0; q < P.q; ++q)
      if (!isfinite(P.mu[q * P.ld_mu + n])) flag |= 1;
    for (int d = 0; d < P.d; ++d) {
      const double y = P.y[d * P.ld_y + n];
      if (!isfinite(y)) flag |= 1;
      yy += y * y;
    }
  }
  if (flag) atomicOr(err, flag);
  red[threadIdx.x] = yy;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void syrk_scalars_kernel(PsiConst P, const double* __restrict__ part, int nb, double* __restrict__ packed) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double yy = 0.0;
  for (int i = 0; i < nb; ++i) yy += part[i];
  packed[0] = double(P.n) * P.variance_d;
  packed[1] = yy;
  packed[2] = double(P.n);
  packed[3] = 0.0;
}

// B operand of the backward GEMM: [2U ; dPsi^T] ((M + D) x M, column-major), split
__global__ void bwd_b_kernel(PsiConst P, int rows, const double* __restrict__ u64, const double* __restrict__ dpsi64,
                             float* __restrict__ big, float* __restrict__ small) {
  const int m = P.m, mv = P.mv;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(rows) * m;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(e % rows), a = int(e / rows);
    const double v = r < m ? 2.0 * u64[r * mv + a] : (r < m + P.d ? dpsi64[int64_t(r - m) * mv + a] : 0.0);
    float b, s;
    split_tf32(v, b, s);
    big[e] = b;
    small[e] = s;
  }
}

// H = G o K and its contractions.  K is read back from the backward chunk matrix as big + small
// (~2^-35 relative, the value the GEMM used); the (x - z) sums are taken as centred moments,
//   sum_n H (x - z)/l = sum H x' - z' sum H,  sum_n H ((x - z)/l)^2 = sum H x'^2 - 2 z' sum H x' + z'^2 sum H
// with x' = (x - c)/l, z' = (z - c)/l and c the mean of Z (P.center): the cancellation is bounded by the
// spread of Z in lengthscales (fp64 keeps ~1e-16 * spread^2).  Lane = inducing point.  Per tile of TR
// rows the block stages K (transposed to [row][a], fp64), G^T ([row][a]) and (x', x'^2) in shared
// memory; the next tile's global loads are issued into registers before the current tile is consumed.
// The 8 warps split the tile's rows; per-lane sums in row order, then the 8 warps in warp order.
// Outputs per slice `by` (before the final 1 / var, 1 / l scalings):
//   oz[q][by][a]          sum_n H (x - z) / l^2
//   os[k][by][blockIdx.x] k = 0: sum H, k = 1 + q: sum H ((x - z) / l)^2, summed over the block's a
//                         in a fixed shuffle tree
constexpr int kRedRows = 1024;
template <int Q>
struct RedTile {
  static constexpr int TR = Q <= 16 ? 64 : 32;     // rows per tile (static shared memory <= 48 KB)
  static constexpr int QC = TR / 4;                // row quads per K column
  static constexpr int KV = TR * 32 / 4 / 256;     // float4 row-quads of K per thread
  static constexpr int GV = TR * 32 / 4 / 256;     // float4 of G^T per thread
  static constexpr int XV = (TR * Q + 255) / 256;  // double2 (x', x'^2) per thread
};
template <int Q>
__global__ void __launch_bounds__(256) syrk_reduce_kernel(PsiConst P, int64_t n0, int64_t nc,
                                                          const float* __restrict__ kbig,
                                                          const float* __restrict__ ksmall,
                                                          const float* __restrict__ gt, int ldg,
                                                          const double2* __restrict__ xp,
                                                          double* __restrict__ oz, double* __restrict__ os) {
  using T = RedTile<Q>;
  constexpr int TR = T::TR;
  __shared__ double s_k[TR][33];
  __shared__ float s_g[TR][32];
  __shared__ double2 s_x[TR * Q];
  __shared__ double red[8][32];
  const int m = P.m, lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int a0 = int(blockIdx.x) * 32, a = a0 + lane;
  const bool va = a < m;
  const int64_t rs = int64_t(blockIdx.y) * kRedRows, re = min(min(nc, P.n - n0), rs + kRedRows);
  // register stage: K as (column al, row quad c), quads fastest -> whole columns per warp, coalesced
  float4 rb[T::KV], rsm[T::KV], rg[T::GV];
  double2 rx[T::XV];
  auto load = [&](int64_t t0) {
#pragma unroll
    for (int i = 0; i < T::KV; ++i) {
      const int e = threadIdx.x + 256 * i, c = e % T::QC, al = e / T::QC;
      const int64_t r = t0 + 4 * c;
      rb[i] = rsm[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (a0 + al < m && r < nc) {
        const int64_t o = r + int64_t(a0 + al) * nc;
        rb[i] = *reinterpret_cast<const float4*>(kbig + o);
        rsm[i] = *reinterpret_cast<const float4*>(ksmall + o);
      }
    }
#pragma unroll
    for (int i = 0; i < T::GV; ++i) {
      const int e = threadIdx.x + 256 * i, c = e & 7, rr = e >> 3;  // 8 quads of a per row
      rg[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t0 + rr < nc && a0 + 4 * c < m) rg[i] = *reinterpret_cast<const float4*>(gt + a0 + 4 * c + (t0 + rr) * ldg);
    }
#pragma unroll
    for (int i = 0; i < T::XV; ++i) {
      const int e = threadIdx.x + 256 * i;
      rx[i] = make_double2(0.0, 0.0);
      if (e < TR * Q && t0 + e / Q < nc) rx[i] = xp[t0 * Q + e];
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int i = 0; i < T::KV; ++i) {
      const int e = threadIdx.x + 256 * i, c = e % T::QC, al = e / T::QC;
      s_k[4 * c + 0][al] = double(rb[i].x) + double(rsm[i].x);
      s_k[4 * c + 1][al] = double(rb[i].y) + double(rsm[i].y);
      s_k[4 * c + 2][al] = double(rb[i].z) + double(rsm[i].z);
      s_k[4 * c + 3][al] = double(rb[i].w) + double(rsm[i].w);
    }
#pragma unroll
    for (int i = 0; i < T::GV; ++i) {
      const int e = threadIdx.x + 256 * i, c = e & 7, rr = e >> 3;
      *reinterpret_cast<float4*>(&s_g[rr][4 * c]) = rg[i];
    }
#pragma unroll
    for (int i = 0; i < T::XV; ++i) {
      const int e = threadIdx.x + 256 * i;
      if (e < TR * Q) s_x[e] = rx[i];
    }
  };
  double mx[Q], m2[Q], dv = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q) mx[q] = m2[q] = 0.0;
  if (rs < re) load(rs);
  for (int64_t t0 = rs; t0 < re; t0 += TR) {
    const int tr = int(min(int64_t(TR), re - t0));
    __syncthreads();
    store();
    __syncthreads();
    if (t0 + TR < re) load(t0 + TR);
#pragma unroll 2
    for (int rr = wp; rr < tr; rr += 8) {
      const double h = double(s_g[rr][lane]) * s_k[rr][lane];
      dv += h;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double2 x = s_x[rr * Q + q];
        mx[q] = fma(h, x.x, mx[q]);
        m2[q] = fma(h, x.y, m2[q]);
      }
    }
  }
  const int64_t nby = gridDim.y, nbx = gridDim.x;
  // the 8 warps' moments for the lane's inducing point, summed in warp order
  auto wsum = [&](double mine) {
    __syncthreads();
    red[wp][lane] = mine;
    __syncthreads();
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][lane];
    return v;
  };
  const double sh = wsum(dv);
  if (wp == 0) {
    const double v = dev::warp_sum_d(va ? sh : 0.0);
    if (lane == 0) os[(int64_t(0) * nby + blockIdx.y) * nbx + blockIdx.x] = v;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double sx = wsum(mx[q]), sx2 = wsum(m2[q]);
    if (wp == 0 && q < P.q) {
      const double zq = va ? (P.z64[a + int64_t(q) * m] - P.center[q]) / P.ls[q] : 0.0;
      if (va) oz[(int64_t(q) * nby + blockIdx.y) * m + a] = (sx - zq * sh) / P.ls[q];
      const double d2 = va ? sx2 - 2.0 * zq * sx + zq * zq * sh : 0.0;
      const double v = dev::warp_sum_d(d2);
      if (lane == 0) os[(int64_t(1 + q) * nby + blockIdx.y) * nbx + blockIdx.x] = v;
    }
  }
}

// grad partial row += the chunk's partials, fixed orders: d Z thread per (a, q) over the slices;
// d var / d l one block per entry over the (slice, a-block) partials.
__global__ void syrk_fold_dz_kernel(int m, int q, int nby, const double* __restrict__ oz, double* __restrict__ acc) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < int64_t(m) * q;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int a = int(i % m), qq = int(i / m);
    double s = 0.0;
    for (int by = 0; by < nby; ++by) s += oz[(int64_t(qq) * nby + by) * m + a];
    acc[1 + q + i] += s;
  }
}
__global__ void __launch_bounds__(256) syrk_fold_sc_kernel(int cnt, const double* __restrict__ os,
                                                           double* __restrict__ acc) {
  __shared__ double red[256];
  const int k = blockIdx.x;  // 0: d var, 1 .. Q: d l
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += os[int64_t(k) * cnt + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) acc[k] += red[0];
}

__global__ void syrk_grads_final_kernel(PsiConst P, const double* __restrict__ acc, double dvar0,
                                        double* __restrict__ packed) {
  const int64_t count = 1 + P.q + int64_t(P.m) * P.q;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < count; k += int64_t(gridDim.x) * blockDim.x) {
    if (k == 0) packed[0] = dvar0 + acc[0] / P.variance_d;
    else if (k <= P.q) packed[k] = acc[k] / P.ls[k - 1];  // sum H ((x - z) / l)^2 / l
    else packed[k] = acc[k];
  }
}

// cuBLAS handle per (host thread, device)
cublasHandle_t handle_for_device() {
  thread_local std::map<int, cublasHandle_t> handles;
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = handles.find(dev);
  if (it != handles.end()) return it->second;
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
  handles[dev] = h;
  return h;
}

// Batched forward: C_i = A_i^T B_i for the nb sub-chunks of kSub rows (A_i = rows of the chunk matrix,
// lda = nc), each the sum of the three split products; fp32 accumulation over kSub rows only.
// The M x M block of C is only ever used symmetrised (syrk_pack_kernel: Phi = (C + C^T) / 2), and there
// small^T big = (big^T small)^T, so it takes two passes: big^T big + 2 big^T small.  The M x D block
// (Psi) keeps all three: big^T big + big^T small + small^T big.
int gemm3_batched_t(cublasHandle_t h, cudaStream_t st, int m, int n, int nb, int nc, const float* big,
                    const float* small, float* c) {
  if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return 3;
  const float one = 1.f, two = 2.f, zero = 0.f;
  const int d = n - m;
  const int64_t cs = int64_t(m) * n, yoff = int64_t(m) * nc;  // batch stride of C, the Y columns of [K | Y]
  auto pass = [&](int cols, const float* a, const float* b, const float* alpha, const float* beta, float* cc) {
    return cublasGemmStridedBatchedEx(h, CUBLAS_OP_T, CUBLAS_OP_N, m, cols, int(kSub), alpha, a, CUDA_R_32F, nc, kSub,
                                      b, CUDA_R_32F, nc, kSub, beta, cc, CUDA_R_32F, m, cs, nb,
                                      CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT) == CUBLAS_STATUS_SUCCESS;
  };
  if (!pass(n, big, big, &one, &zero, c)) return 3;              // big^T [big | big_Y]
  if (!pass(m, big, small, &two, &one, c)) return 3;             // + 2 big^T small   (Phi block)
  if (d > 0) {
    if (!pass(d, big, small + yoff, &one, &one, c + int64_t(m) * m)) return 3;  // + big^T small_Y
    if (!pass(d, small, big + yoff, &one, &one, c + int64_t(m) * m)) return 3;  // + small^T big_Y
  }
  g_tc_launches.fetch_add(d > 0 ? 4 : 2);
  return 0;
}

// C (+)= sum of the three split products op(A) B: big.big + big.small + small.big (TF32 tensor cores)
int gemm3(cublasHandle_t h, cudaStream_t st, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k,
          const float* abig,
          const float* asmall, int lda, const float* bbig, const float* bsmall, int ldb, float* c, int ldc) {
  if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return 3;
  const float one = 1.f, zero = 0.f;
  const float* as[3] = {abig, abig, asmall};
  const float* bs[3] = {bbig, bsmall, bbig};
  for (int i = 0; i < 3; ++i) {
    if (cublasGemmEx(h, ta, tb, m, n, k, &one, as[i], CUDA_R_32F, lda, bs[i], CUDA_R_32F, ldb,
                     i == 0 ? &zero : &one, c, CUDA_R_32F, ldc, CUBLAS_COMPUTE_32F_FAST_TF32,
                     CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
      return 3;
  }
  g_tc_launches.fetch_add(3);
  return 0;
}

constexpr int kSyrkQs[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 48, 64};
int syrk_q(int q) {
  for (int v : kSyrkQs)
    if (v >= q) return v;
  return -1;
}

inline int bwd_k(const PsiConst& P) { return (P.m + P.d + 3) / 4 * 4; }  // chunk-matrix columns, 16-byte rows
inline int bwd_ldg(const PsiConst& P) { return (P.m + 3) / 4 * 4; }
inline int64_t rows_pad(const PsiConst& P) { return (P.n + kSub - 1) / kSub * kSub; }

// The forward's split Knm tiles are kept for the backward (one less exp pass per evaluation) while
// they fit the budget: N x (M + D) x 8 bytes + the (x', x'^2) rows; 64 GiB by default (the C4 shape
// at N = 10M takes 41 GB of the 180 GB), SGPX_SYRK_CACHE_GIB overrides (0 = always recompute).
// A pure function of the shapes, so the forward and backward plans agree.
bool syrk_cached(const PsiConst& P) {
  double gib = 64.0;
  if (const char* e = getenv("SGPX_SYRK_CACHE_GIB")) gib = atof(e);
  const double bytes = double(rows_pad(P)) * (double(bwd_k(P)) * 8.0 + double(syrk_q(P.q)) * 16.0);
  return bytes <= gib * 1073741824.0;
}

// Forward region (the backward reads its cache through BwdConst::fwd_rt): [big | small | xp] first,
// sized for all rows when cached, else one chunk each (xp unused); then the batched GEMM output,
// the fp64 accumulator and the per-row scalars.
struct SyrkFwd {
  int64_t ncols, off_big, off_small, off_xp, off_c, off_acc, off_rows, doubles;
  int nrb;
  bool cached;
};
SyrkFwd fwd_layout(const PsiConst& P, int num_sms) {
  SyrkFwd L{};
  L.cached = syrk_cached(P);
  L.ncols = bwd_k(P);
  const int64_t rows = L.cached ? rows_pad(P) : kChunk;
  const int64_t mat_doubles = (rows * L.ncols + 1) / 2 / 2 * 2 + 2;  // floats -> doubles, 16-byte multiple
  L.off_big = 0;
  L.off_small = L.off_big + mat_doubles;
  L.off_xp = L.off_small + mat_doubles;
  L.off_c = L.off_xp + (L.cached ? 2 * rows * syrk_q(P.q) : 0);
  L.off_acc = L.off_c + (int64_t(kBatch) * P.m * (P.m + P.d) + 1) / 2;
  L.off_rows = L.off_acc + int64_t(P.m) * (P.m + P.d);
  L.nrb = int(std::max<int64_t>(1, std::min<int64_t>((P.n + 255) / 256, 2 * int64_t(num_sms))));
  L.doubles = L.off_rows + L.nrb + 4;
  return L;
}

struct SyrkBwd {
  int64_t off_abig, off_asmall, off_bbig, off_bsmall, off_g, off_rows, off_os, off_acc, off_xp, doubles;
  int nby;
};
SyrkBwd bwd_layout(const PsiConst& P, int q) {
  SyrkBwd L{};
  const int64_t k = bwd_k(P);
  const bool own = !syrk_cached(P);  // the chunk matrices and x' rows, when the forward keeps none
  L.nby = int((kChunk + kRedRows - 1) / kRedRows);
  L.off_abig = 0;
  L.off_asmall = L.off_abig + (own ? (kChunk * k + 1) / 2 : 0);
  L.off_bbig = L.off_asmall + (own ? (kChunk * k + 1) / 2 : 0);
  L.off_bsmall = L.off_bbig + (k * P.m + 1) / 2;
  L.off_g = L.off_bsmall + (k * P.m + 1) / 2;
  L.off_rows = L.off_g + (kChunk * bwd_ldg(P) + 1) / 2;
  L.off_os = L.off_rows + int64_t(L.nby) * P.m * q;  // oz (Q x nby x M), then os ((1 + Q) x nby x nbx)
  L.off_acc = L.off_os + int64_t(1 + q) * L.nby * ((P.m + 31) / 32);
  L.off_xp = (L.off_acc + 1 + P.q + int64_t(P.m) * P.q + 1) / 2 * 2;  // 16-byte aligned
  L.doubles = L.off_xp + (own ? 2 * kChunk * q : 0) + 4;
  return L;
}

float* as_floats(double* p) { return reinterpret_cast<float*>(p); }


template <int Q>
int syrk_backward_q(const PsiConst& P, const BwdConst& B, double* base, double* packed, int num_sms,
                    cudaStream_t st) {
  const SyrkBwd L = bwd_layout(P, Q);
  cublasHandle_t h = handle_for_device();
  if (!h) return 3;
  const int k = bwd_k(P);
  const int bb = int(std::min<int64_t>((int64_t(k) * P.m + 255) / 256, int64_t(num_sms) * 8));
  bwd_b_kernel<<<bb, 256, 0, st>>>(P, k, B.u64, B.dpsi64, as_floats(base + L.off_bbig), as_floats(base + L.off_bsmall));
  double* acc = base + L.off_acc;
  const int64_t count = 1 + P.q + int64_t(P.m) * P.q;
  cudaMemsetAsync(acc, 0, sizeof(double) * count, st);
  g_tc_launches.fetch_add(1);
  const bool cached = syrk_cached(P);
  double* fbase = const_cast<double*>(B.fwd_rt);
  const SyrkFwd F = fwd_layout(P, num_sms);
  for (int64_t n0 = 0; n0 < P.n; n0 += kChunk) {
    float *kb, *ks;
    double2* xp;
    int64_t nc;
    if (cached) {  // the forward's tiles: its chunk geometry (whole kSub sub-chunks)
      nc = std::min<int64_t>(kChunk, (P.n - n0 + kSub - 1) / kSub * kSub);
      kb = as_floats(fbase + F.off_big) + n0 * k;
      ks = as_floats(fbase + F.off_small) + n0 * k;
      xp = reinterpret_cast<double2*>(fbase + F.off_xp) + n0 * Q;
    } else {
      nc = std::min<int64_t>(kChunk, (P.n - n0 + 3) / 4 * 4);
      kb = as_floats(base + L.off_abig);
      ks = as_floats(base + L.off_asmall);
      xp = reinterpret_cast<double2*>(base + L.off_xp);
      knm_split_kernel<Q><<<dim3(unsigned((nc + 255) / 256), unsigned((k + kCols - 1) / kCols)), 256, 0, st>>>(
          P, n0, nc, k, kb, ks, xp);
      g_tc_launches.fetch_add(1);
    }
    // G^T (M x nc) = [2U ; dPsi^T ; 0]^T (M x k) . [K | Y | 0]^T (k x nc)
    const int ldg = bwd_ldg(P);
    if (gemm3(h, st, CUBLAS_OP_T, CUBLAS_OP_T, P.m, int(nc), k, as_floats(base + L.off_bbig),
              as_floats(base + L.off_bsmall), k, kb, ks, int(nc), as_floats(base + L.off_g), ldg))
      return 3;
    const int nby = int((nc + kRedRows - 1) / kRedRows);
    const int nbx = (P.m + 31) / 32;
    syrk_reduce_kernel<Q><<<dim3(unsigned(nbx), unsigned(nby)), 256, 0, st>>>(
        P, n0, nc, kb, ks, as_floats(base + L.off_g), ldg, xp, base + L.off_rows, base + L.off_os);
    syrk_fold_dz_kernel<<<int(std::min<int64_t>((int64_t(P.m) * P.q + 255) / 256, 256)), 256, 0, st>>>(
        P.m, P.q, nby, base + L.off_rows, acc);
    syrk_fold_sc_kernel<<<1 + P.q, 256, 0, st>>>(nby * nbx, base + L.off_os, acc);
    g_tc_launches.fetch_add(3);
  }
  syrk_grads_final_kernel<<<int(std::min<int64_t>((count + 255) / 256, 256)), 256, 0, st>>>(
      P, acc, B.d_phi * double(P.n), packed);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int Q>
int syrk_forward_q(const PsiConst& P, double* base, double* packed, int* err_flag, int num_sms, cudaStream_t st) {
  const SyrkFwd L = fwd_layout(P, num_sms);
  cublasHandle_t h = handle_for_device();
  if (!h) return 3;
  double* acc = base + L.off_acc;
  const int64_t ccount = int64_t(P.m) * (P.m + P.d);
  cudaMemsetAsync(acc, 0, sizeof(double) * ccount, st);
  syrk_rows_kernel<<<L.nrb, 256, 0, st>>>(P, base + L.off_rows, err_flag);
  g_tc_launches.fetch_add(1);
  for (int64_t n0 = 0; n0 < P.n; n0 += kChunk) {
    // whole sub-chunks (zero rows past N contribute nothing)
    const int64_t nc = std::min<int64_t>(kChunk, (P.n - n0 + kSub - 1) / kSub * kSub);
    const int nb = int(nc / kSub);
    float* kb = as_floats(base + L.off_big) + (L.cached ? n0 * L.ncols : 0);
    float* ks = as_floats(base + L.off_small) + (L.cached ? n0 * L.ncols : 0);
    double2* xp = L.cached ? reinterpret_cast<double2*>(base + L.off_xp) + n0 * Q : nullptr;
    knm_split_kernel<Q><<<dim3(unsigned((nc + 255) / 256), unsigned((L.ncols + kCols - 1) / kCols)), 256, 0, st>>>(
        P, n0, nc, int(L.ncols), kb, ks, xp);
    g_tc_launches.fetch_add(1);
    // C_i (M x (M + D)) = K_i^T [K_i | Y_i] per sub-chunk i: A = the first M columns of the chunk matrix
    if (gemm3_batched_t(h, st, P.m, P.m + P.d, nb, int(nc), kb, ks, as_floats(base + L.off_c))) return 3;
    acc_add_kernel<<<int(std::min<int64_t>((ccount + 255) / 256, 1024)), 256, 0, st>>>(
        acc, as_floats(base + L.off_c), nb, ccount);
    g_tc_launches.fetch_add(1);
  }
  const int64_t npairs = int64_t(P.m) * (P.m + 1) / 2;
  syrk_pack_kernel<<<int(std::min<int64_t>((npairs + int64_t(P.m) * P.d + 255) / 256, 1024)), 256, 0, st>>>(P, acc,
                                                                                                           packed);
  syrk_scalars_kernel<<<1, 32, 0, st>>>(P, base + L.off_rows, L.nrb, packed);
  g_tc_launches.fetch_add(2);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

bool syrk_supported(const PsiConst& P) { return !P.expected && syrk_q(P.q) > 0 && P.m >= 1; }
int64_t syrk_fwd_doubles(const PsiConst& P, int num_sms) { return fwd_layout(P, num_sms).doubles; }
int64_t syrk_bwd_doubles(const PsiConst& P, int num_sms) {
  (void)num_sms;
  return bwd_layout(P, std::max(1, syrk_q(P.q))).doubles;
}

#define SGPX_SYRK_DISPATCH(fn, ...)     \
  switch (syrk_q(P.q)) {                \
    case 1: return fn<1>(__VA_ARGS__);  \
    case 2: return fn<2>(__VA_ARGS__);  \
    case 3: return fn<3>(__VA_ARGS__);  \
    case 4: return fn<4>(__VA_ARGS__);  \
    case 5: return fn<5>(__VA_ARGS__);  \
    case 6: return fn<6>(__VA_ARGS__);  \
    case 8: return fn<8>(__VA_ARGS__);  \
    case 10: return fn<10>(__VA_ARGS__); \
    case 12: return fn<12>(__VA_ARGS__); \
    case 16: return fn<16>(__VA_ARGS__); \
    case 20: return fn<20>(__VA_ARGS__); \
    case 24: return fn<24>(__VA_ARGS__); \
    case 32: return fn<32>(__VA_ARGS__); \
    case 48: return fn<48>(__VA_ARGS__); \
    case 64: return fn<64>(__VA_ARGS__); \
    default: return 1;                   \
  }

int syrk_forward(const PsiConst& P, double* base, double* packed, int* err_flag, int num_sms, void* stream) {
  SGPX_SYRK_DISPATCH(syrk_forward_q, P, base, packed, err_flag, num_sms, static_cast<cudaStream_t>(stream))
}

int syrk_backward(const PsiConst& P, const BwdConst& B, double* base, double* packed, int num_sms, void* stream) {
  SGPX_SYRK_DISPATCH(syrk_backward_q, P, B, base, packed, num_sms, static_cast<cudaStream_t>(stream))
}

}  // namespace sgpx
