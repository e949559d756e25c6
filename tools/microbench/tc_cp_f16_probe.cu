// tc_cp_f16_probe.cu -- checks the MMA1 scheme of the row-tile kernel on hardware:
//   1. tcgen05.cp.128x256b copies a canonical K-major (no swizzle) [128 x 16 u32] shared-memory
//      tile into TMEM (lane = row, column = u32 index), 8 columns per instruction;
//   2. kind::f16 MMA with A = packed half2 in TMEM (low half = even k) and B = fp16 canonical
//      K-major in shared memory computes D = A B^T;
//   3. the 3-piece split hi*hi + hi*lo + lo*hi of fp32 features reaches ~2^-22 relative accuracy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_cp_f16_probe tc_cp_f16_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../paper_1410_4984_b200/csrc/tc_util.cuh"

using namespace sgpx;

constexpr int KH = 32;       // halves per piece
constexpr int NB = 96;       // B rows
constexpr int KU = KH / 2;   // u32 per piece row

__device__ __forceinline__ int canon_u32(int r, int j, int kdim_u32) {
  return (r >> 3) * (kdim_u32 * 8) + (j >> 2) * 32 + (r & 7) * 4 + (j & 3);
}

__global__ void probe(const uint32_t* a_hi, const uint32_t* a_lo, const uint32_t* b_hi, const uint32_t* b_lo,
                      float* d_out, uint32_t* cp_out) {
  __shared__ __align__(1024) uint32_t sa[2][128 * KU];
  __shared__ __align__(1024) uint32_t sb[2][NB * KU];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * KU; i += blockDim.x) {
    const int r = i / KU, j = i % KU;
    sa[0][canon_u32(r, j, KU)] = a_hi[i];
    sa[1][canon_u32(r, j, KU)] = a_lo[i];
  }
  for (int i = tid; i < NB * KU; i += blockDim.x) {
    const int r = i / KU, j = i % KU;
    sb[0][canon_u32(r, j, KU)] = b_hi[i];
    sb[1][canon_u32(r, j, KU)] = b_lo[i];
  }
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  asm volatile("fence.proxy.async.shared::cta;");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  const uint32_t ta = tmem + 256;  // A: hi cols [256, 272), lo cols [272, 288)
  if (warp == 0) {
    // copy A hi / lo: 8 u32 columns (two core matrices along K) per instruction
    for (int p = 0; p < 2; ++p)
      for (int c = 0; c < KU / 8; ++c) {
        const uint64_t sd = tc::desc(tc::smem_u32(&sa[p][0]) + 256u * c, KU);
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(ta + uint32_t(p * KU + 8 * c)),
            "l"(sd));
      }
    const uint32_t id = (1u << 4) | (uint32_t(NB >> 3) << 17) | (uint32_t(128 >> 4) << 24);  // f16 x f16 -> f32
    int first = 1;
    for (int t = 0; t < 3; ++t) {  // hi*hi, hi*lo, lo*hi
      const uint32_t a = ta + (t == 2 ? KU : 0);
      const uint32_t bs = tc::smem_u32(&sb[t == 1 ? 1 : 0][0]);
      for (int s = 0; s < KH / 16; ++s) {
        const uint64_t bd = tc::desc(bs + 256u * s, KU);
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
            "r"(a + 8u * s), "l"(bd), "r"(id), "r"(first ? 0u : 1u));
        first = 0;
      }
    }
    tc::commit_w(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  if (warp < 4) {
    const int row = 32 * warp + lane;
    const uint32_t lo = uint32_t(32 * warp) << 16;
    for (int c0 = 0; c0 < NB; c0 += 16) {
      uint32_t r[16];
      tc::ld16(tmem + lo + c0, r);
      tc::ld_wait();
      for (int i = 0; i < 16; ++i) d_out[row * NB + c0 + i] = __uint_as_float(r[i]);
    }
    uint32_t r[16];
    tc::ld16(ta + lo, r);
    tc::ld_wait();
    for (int i = 0; i < 16; ++i) cp_out[row * 32 + i] = r[i];
    tc::ld16(ta + lo + 16, r);
    tc::ld_wait();
    for (int i = 0; i < 16; ++i) cp_out[row * 32 + 16 + i] = r[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

static void split(float x, __half& h, __half& l) {
  h = __float2half_rn(x);
  l = __float2half_rn(x - __half2float(h));
}
static uint32_t pack(__half lo_k, __half hi_k) {
  return uint32_t(*reinterpret_cast<uint16_t*>(&lo_k)) | (uint32_t(*reinterpret_cast<uint16_t*>(&hi_k)) << 16);
}

int main() {
  srand(1);
  static float A[128][KH], B[NB][KH];
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < KH; ++k) A[r][k] = k < 22 ? (rand() / float(RAND_MAX) - 0.5f) * (k == 21 ? 40.f : 4.f) : 0.f;
  for (int r = 0; r < NB; ++r)
    for (int k = 0; k < KH; ++k) B[r][k] = k < 22 ? (rand() / float(RAND_MAX) - 0.5f) * 3.f : 0.f;
  static uint32_t ah[128 * KU], al[128 * KU], bh[NB * KU], bl[NB * KU];
  for (int r = 0; r < 128; ++r)
    for (int j = 0; j < KU; ++j) {
      __half h0, l0, h1, l1;
      split(A[r][2 * j], h0, l0);
      split(A[r][2 * j + 1], h1, l1);
      ah[r * KU + j] = pack(h0, h1);
      al[r * KU + j] = pack(l0, l1);
    }
  for (int r = 0; r < NB; ++r)
    for (int j = 0; j < KU; ++j) {
      __half h0, l0, h1, l1;
      split(B[r][2 * j], h0, l0);
      split(B[r][2 * j + 1], h1, l1);
      bh[r * KU + j] = pack(h0, h1);
      bl[r * KU + j] = pack(l0, l1);
    }
  uint32_t *dah, *dal, *dbh, *dbl, *dcp;
  float* dd;
  cudaMalloc(&dah, sizeof(ah));
  cudaMalloc(&dal, sizeof(al));
  cudaMalloc(&dbh, sizeof(bh));
  cudaMalloc(&dbl, sizeof(bl));
  cudaMalloc(&dd, 128 * NB * 4);
  cudaMalloc(&dcp, 128 * 32 * 4);
  cudaMemcpy(dah, ah, sizeof(ah), cudaMemcpyHostToDevice);
  cudaMemcpy(dal, al, sizeof(al), cudaMemcpyHostToDevice);
  cudaMemcpy(dbh, bh, sizeof(bh), cudaMemcpyHostToDevice);
  cudaMemcpy(dbl, bl, sizeof(bl), cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dah, dal, dbh, dbl, dd, dcp);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  static float D[128 * NB];
  static uint32_t cp[128 * 32];
  cudaMemcpy(D, dd, sizeof(D), cudaMemcpyDeviceToHost);
  cudaMemcpy(cp, dcp, sizeof(cp), cudaMemcpyDeviceToHost);
  int cp_bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int j = 0; j < KU; ++j) {
      if (cp[r * 32 + j] != ah[r * KU + j]) ++cp_bad;
      if (cp[r * 32 + KU + j] != al[r * KU + j]) ++cp_bad;
    }
  double max_err = 0, max_abs = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < NB; ++n) {
      double ref = 0, mag = 0;
      for (int k = 0; k < KH; ++k) {
        ref += double(A[r][k]) * double(B[n][k]);
        mag += fabs(double(A[r][k]) * double(B[n][k]));
      }
      const double err = fabs(D[r * NB + n] - ref) / mag;
      max_err = err > max_err ? err : max_err;
      max_abs = fabs(D[r * NB + n] - ref) > max_abs ? fabs(D[r * NB + n] - ref) : max_abs;
    }
  printf("tcgen05.cp mismatches: %d of %d\n", cp_bad, 128 * KH);
  printf("3-piece fp16 MMA: max error / sum|terms| = %.3e (2^-22 = %.3e), max abs %.3e\n", max_err,
         std::ldexp(1.0, -22), max_abs);
  return (cp_bad == 0 && max_err < 4 * std::ldexp(1.0, -22)) ? 0 : 1;
}
