// psi_common.cuh -- device helpers shared by the SIMT and the tensor-core psi kernels:
// per-datapoint tables (psi_stats.hpp:144-167 restated with the exponent factorisation of
// DESIGN.md §3), L_na, warp reduce-scatters.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

#include "psi_kernels.cuh"

namespace sgpx {
namespace dev {

constexpr float kLog2e = 1.4426950408889634f;
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (offloads MUFU.EX2, which is 16/clk/SM): round-to-nearest split x = j + f,
// f in [-1/2, 1/2], degree-5 relative-minimax polynomial (max rel. error 2.0e-7 in fp32 Horner,
// on par with ex2.approx), exponent added with one integer op.  x is clamped at -125 (returns
// ~2^-125 instead of 0 for -inf; harmless in sums).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: round(x) lands in the low mantissa bits
  const float f = x - (t - 12582912.f);
  float p = fmaf(0.001328189391642809f, f, 0.009675598703324795f);
  p = fmaf(p, f, 0.05550696700811386f);
  p = fmaf(p, f, 0.24022118747234344f);
  p = fmaf(p, f, 0.6931470036506653f);
  p = fmaf(p, f, 1.0000001192092896f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ int64_t pair_index(int a, int b, int m) {
  // upper triangle, m1-major order (psi_stats.hpp:85-97)
  return int64_t(a) * (2 * m - a + 1) / 2 + (b - a);
}

// Per-chunk per-datapoint tables, each [qv][32] (lane-contiguous) unless noted.
struct Rows {
  float *mu, *d1, *d2, *sv, *al, *be, *kk, *t1, *t2, *b1, *b2;
};

__host__ __device__ inline int rows_floats(int qv) { return 9 * qv * 32 + 64; }

__device__ __forceinline__ Rows carve_rows(float*& p, int qv) {
  Rows r;
  const int sz = qv * 32;
  r.mu = p; p += sz;
  r.d1 = p; p += sz;
  r.d2 = p; p += sz;
  r.sv = p; p += sz;
  r.al = p; p += sz;
  r.be = p; p += sz;
  r.kk = p; p += sz;
  r.t1 = p; p += sz;
  r.t2 = p; p += sz;
  r.b1 = p; p += 32;
  r.b2 = p; p += 32;
  return r;
}

template <int Q>
__device__ __forceinline__ void load_z(const float* src, float (&z)[Q]) {
  constexpr int Q4 = (Q + 3) / 4;
#pragma unroll
  for (int i = 0; i < Q4; ++i) {
    const float4 t = reinterpret_cast<const float4*>(src)[i];
    if (4 * i + 0 < Q) z[(4 * i + 0) % Q] = t.x;
    if (4 * i + 1 < Q) z[(4 * i + 1) % Q] = t.y;
    if (4 * i + 2 < Q) z[(4 * i + 2) % Q] = t.z;
    if (4 * i + 3 < Q) z[(4 * i + 3) % Q] = t.w;
  }
}

// Per-datapoint constants of psi_stats.hpp:144-167, fp64 in -> fp32 tables, with
// the translation by P.center.  Validation of psi_stats.hpp:119-120 is fused
// (err_flag bit 0).  kl_acc (latent engine): KL partial of parallel.hpp:148-149.
template <int Q>
__device__ void load_rows(const PsiConst& P, int64_t n0, const Rows& R, double* kl_acc, int* err_flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t n = n0 + lane;
  const bool valid = n < P.n;
  for (int q = warp; q < P.qv; q += nw) {
    float mu = 0.f, sv = 0.f, d1 = 0.f, d2 = 0.f, al = 0.f, be = 0.f, kk = 0.f, t1 = 0.f, t2 = 0.f;
    if (q < P.q && valid) {
      const double mud = P.mu[q * P.ld_mu + n];
      const double sd = P.expected ? P.s[q * P.ld_s + n] : 0.0;
      if (err_flag && !isfinite(mud)) atomicOr(err_flag, 1);
      if (err_flag && P.expected && !(sd > 0.0 && isfinite(sd))) atomicOr(err_flag, 4);
      if (kl_acc) *kl_acc += 0.5 * (sd + mud * mud - log(sd) - 1.0);
      mu = float(mud - P.center[q]);
      sv = float(sd);
      const float l2 = P.l2[q], il2 = P.il2[q];
      d1 = 1.f / (sv + l2);
      d2 = 1.f / (2.f * sv + l2);
      al = kLog2e * d2 * mu;
      be = -0.25f * kLog2e * (il2 + d2);
      kk = kLog2e * sv * il2 * d2;  // = log2e (1/l^2 - d2)/2 without cancellation
      t1 = -0.5f * log2f(1.f + sv * il2);
      t2 = -0.5f * log2f(1.f + 2.f * sv * il2) - kLog2e * d2 * mu * mu;
    }
    const int i = q * 32 + lane;
    R.mu[i] = mu;
    R.d1[i] = d1;
    R.d2[i] = d2;
    R.sv[i] = sv;
    R.al[i] = al;
    R.be[i] = be;
    R.kk[i] = kk;
    R.t1[i] = t1;
    R.t2[i] = t2;
  }
  __syncthreads();
  if (warp == 0) {
    float b1 = P.log2_var, b2 = 2.f * P.log2_var;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      b1 += R.t1[q * 32 + lane];
      b2 += R.t2[q * 32 + lane];
    }
    R.b1[lane] = valid ? b1 : -CUDART_INF_F;
    R.b2[lane] = valid ? b2 : -CUDART_INF_F;
  }
  __syncthreads();
}

// L'_na = sum_q (al z + be z^2) + B_n/2 for every inducing index a (padded rows -inf).
template <int Q>
__device__ __forceinline__ void build_L(const PsiConst& P, const Rows& R, const float* Zc, float* Ls) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float al[Q], be[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    al[q] = R.al[q * 32 + lane];
    be[q] = R.be[q * 32 + lane];
  }
  const float bh = 0.5f * R.b2[lane];
  for (int a = warp; a < P.mv; a += nw) {
    float L = -CUDART_INF_F;
    if (a < P.m) {
      float z[Q];
      load_z<Q>(Zc + a * P.qv, z);
      L = bh;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        L = fmaf(al[q], z[q], L);
        L = fmaf(be[q] * z[q], z[q], L);
      }
    }
    Ls[a * 32 + lane] = L;
  }
}

// Sum of v[lane>>1] over the warp, for 16 values per lane (lanes 2k, 2k+1 hold index k).
__device__ __forceinline__ float reduce_scatter16(float (&v)[16], int lane) {
  bool h = lane & 16;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float send = h ? v[i] : v[i + 8];
    const float keep = h ? v[i + 8] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  h = lane & 8;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = h ? v[i] : v[i + 4];
    const float keep = h ? v[i + 4] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  h = lane & 4;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = h ? v[i] : v[i + 2];
    const float keep = h ? v[i + 2] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  h = lane & 2;
  {
    const float send = h ? v[0] : v[1];
    const float keep = h ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Sum of v[lane] over the warp, 32 values per lane.
__device__ __forceinline__ float reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
  for (int half = 16; half >= 1; half >>= 1) {
    const bool h = lane & half;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = h ? v[i] : v[i + half];
      const float keep = h ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  return v[0];
}

// Sum of v[i] over the warp for K values per lane (K in {8, 16, 32}): lane ends up holding
// the total of index lane >> (5 - log2 K).
template <int K>
__device__ __forceinline__ float reduce_scatter(float (&v)[K], int lane) {
  int n = K;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (n > 1) {
      const int h = n >> 1;
      const bool hi = lane & off;
#pragma unroll
      for (int i = 0; i < K / 2; ++i) {
        if (i < h) {
          const float send = hi ? v[i] : v[i + h];
          const float keep = hi ? v[i + h] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      n = h;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  return v[0];
}

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}


}  // namespace dev
}  // namespace sgpx
