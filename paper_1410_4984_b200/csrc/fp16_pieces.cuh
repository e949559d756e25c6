// fp16_pieces.cuh -- 16-bit piece splits and the canonical K-major feature-row layout shared by the
// row-tile psi2 kernels (psi_rowtile.cu) and the tcgen05 psi1 kernels (psi1_tc.cu).
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

namespace sgpx {
namespace pc {

constexpr float kHalfMax = 6.0e4f;  // exponent features are clamped to the fp16 range

// fp16 hi / lo split of two floats: hi = f16x2(a, b), lo = f16x2(a - hi.a, b - hi.b).  Written with the
// packed cvt and a b16 split so ptxas reads the halves with HADD2.F32 .H0 / .H1 selectors (3
// instructions per value; the __half2 intrinsics cost ~2 extra PRMT per value).
__device__ __forceinline__ void split_f16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  uint32_t h;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));
  float ha, hb;
  asm("{.reg .b16 l, u; mov.b32 {l, u}, %2; cvt.f32.f16 %0, l; cvt.f32.f16 %1, u;}" : "=f"(ha), "=f"(hb) : "r"(h));
  uint32_t l2;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l2) : "f"(b - hb), "f"(a - ha));
  hi = h;
  lo = l2;
}

__device__ __forceinline__ uint32_t h2u(__half2 h) {
  return uint32_t(__half_as_ushort(__low2half(h))) | (uint32_t(__half_as_ushort(__high2half(h))) << 16);
}

// fp16 pieces of features k, k+1 packed as half2 words (low half = even k), clamped to the fp16
// range: NP = 2 -> hi, lo (~2^-22); NP = 3 -> hi, mid, lo (~2^-33, from fp64 features)
template <int NP>
__device__ __forceinline__ void split_pair(double x0, double x1, uint32_t (&w)[NP]) {
  x0 = fmin(fmax(x0, -double(kHalfMax)), double(kHalfMax));
  x1 = fmin(fmax(x1, -double(kHalfMax)), double(kHalfMax));
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const __half2 h = __floats2half2_rn(float(x0), float(x1));
    w[i] = h2u(h);
    const float2 hf = __half22float2(h);
    x0 -= double(hf.x);
    x1 -= double(hf.y);
  }
}
// 2 K1 features of one row as NP pieces of K1 words at word offset `row_off` of a canonical
// K-major tile (core matrix = 8 rows x 4 words); piece i at base + i * pstride
template <int NP>
__device__ __forceinline__ void put_feat_words(float* base, int64_t pstride, int64_t row_off, const double* f, int K1) {
  for (int k = 0; k < K1; k += 4) {
    uint32_t w[4][NP];
#pragma unroll
    for (int u = 0; u < 4; ++u) split_pair<NP>(f[2 * (k + u)], f[2 * (k + u) + 1], w[u]);
#pragma unroll
    for (int i = 0; i < NP; ++i)
      *reinterpret_cast<uint4*>(base + i * pstride + row_off + (k >> 2) * 32) = make_uint4(w[0][i], w[1][i], w[2][i], w[3][i]);
  }
}
template <int NP>
__device__ __forceinline__ void put_rows(float* base, int64_t pstride, int64_t r, const double* f, int K1) {
  put_feat_words<NP>(base, pstride, (r >> 3) * (K1 * 8) + (r & 7) * 4, f, K1);
}

}  // namespace pc
}  // namespace sgpx
