// 32 x 32 in-warp Cholesky variants (the diagonal blocks of bound_g_small_kernel): cycles per factorisation.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int M = 100;
// V1: shared memory, lane = row, 4-wide updates (the current kernel)
__device__ void fac_smem(double* Lp, int m, int jb, double* invd) {
  const int r = threadIdx.x & 31;
  for (int k = 0; k < jb; ++k) {
    const double dkk = Lp[k + k * m];
    const double inv = rsqrt(dkk), lkk = dkk * inv;
    double lrk = 0.0;
    if (r > k && r < jb) { lrk = Lp[r + k * m] * inv; Lp[r + k * m] = lrk; }
    if (r == k) { Lp[k + k * m] = lkk; invd[k] = inv; }
    __syncwarp();
    if (r > k && r < jb) {
      int c = k + 1;
      for (; c + 3 <= r; c += 4) {
        const double l0 = Lp[c + k * m], l1 = Lp[c + 1 + k * m], l2 = Lp[c + 2 + k * m], l3 = Lp[c + 3 + k * m];
        const double a0 = Lp[r + c * m], a1 = Lp[r + (c + 1) * m], a2 = Lp[r + (c + 2) * m], a3 = Lp[r + (c + 3) * m];
        Lp[r + c * m] = fma(-lrk, l0, a0); Lp[r + (c + 1) * m] = fma(-lrk, l1, a1);
        Lp[r + (c + 2) * m] = fma(-lrk, l2, a2); Lp[r + (c + 3) * m] = fma(-lrk, l3, a3);
      }
      for (; c <= r; ++c) Lp[r + c * m] = fma(-lrk, Lp[c + k * m], Lp[r + c * m]);
    }
    __syncwarp();
  }
}
// V3: shared memory, lane = row; per step every candidate column loaded first (predicated, compile-time
// indices in halves of 16), then the FMAs, then the stores -- no load waits behind an earlier store
__device__ void fac_smem_batched(double* Lp, int m, int jb, double* invd) {
  const int r = threadIdx.x & 31;
  for (int k = 0; k < jb; ++k) {
    const double dkk = Lp[k + k * m];
    const double inv = rsqrt(dkk), lkk = dkk * inv;
    double lrk = 0.0;
    if (r > k && r < jb) { lrk = Lp[r + k * m] * inv; Lp[r + k * m] = lrk; }
    if (r == k) { Lp[k + k * m] = lkk; invd[k] = inv; }
    __syncwarp();
    const bool rowact = r > k && r < jb;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (16 * h + 15 <= k) continue;  // warp-uniform
      double a[16], l[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int c = 16 * h + u;
        const bool act = rowact && c > k && c <= r;
        a[u] = act ? Lp[r + c * m] : 0.0;
        l[u] = act ? Lp[c + k * m] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int c = 16 * h + u;
        if (rowact && c > k && c <= r) Lp[r + c * m] = fma(-lrk, l[u], a[u]);
      }
    }
    __syncwarp();
  }
}
// V2: registers, lane = row, every warp (converged), shuffles; writes by warp 0
__device__ void fac_reg(double* Lp, int m, double* invd) {
  const int r = threadIdx.x & 31;
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = Lp[r + c * m];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double dkk = __shfl_sync(0xffffffffu, row[k], k);
    const double inv = rsqrt(dkk), lkk = dkk * inv;
    const double lrk = r > k ? row[k] * inv : 0.0;
    row[k] = r > k ? lrk : (r == k ? lkk : 0.0);
    if (r == k && threadIdx.x < 32) invd[k] = inv;
#pragma unroll
    for (int c = k + 1; c < 32; ++c) {
      const double lck = __shfl_sync(0xffffffffu, lrk, c);
      row[c] = r >= c ? fma(-lrk, lck, row[c]) : row[c];
    }
  }
  __syncthreads();
  if (threadIdx.x < 32)
#pragma unroll
    for (int c = 0; c < 32; ++c) if (c <= r) Lp[r + c * m] = row[c];
}
template <int V>
__global__ void __launch_bounds__(512) kern(const double* a, long long* t, double* out) {
  extern __shared__ double sm[];
  __shared__ double invd[32];
  for (int e = threadIdx.x; e < M * M; e += blockDim.x) sm[e] = a[e];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 3; ++rep) {
    if (V == 1) {
      if (threadIdx.x < 32) fac_smem(sm, M, 32, invd);
      __syncthreads();
    } else if (V == 3) {
      if (threadIdx.x < 32) fac_smem_batched(sm, M, 32, invd);
      __syncthreads();
    } else {
      fac_reg(sm, M, invd);
      __syncthreads();
    }
    for (int e = threadIdx.x; e < M * M; e += blockDim.x) sm[e] = a[e];  // restore
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *t = (t1 - t0) / 3;
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) out[e] = sm[(e % 32) + (e / 32) * M];
}
int main() {
  double h[M * M];
  for (int i = 0; i < M; ++i) for (int j = 0; j < M; ++j) h[i + j * M] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + (i - j) * (i - j));
  double *a, *o1, *o2; long long* t; cudaMalloc(&a, sizeof(h)); cudaMalloc(&o1, 8192); cudaMalloc(&o2, 8192); cudaMallocManaged(&t, 16);
  cudaMemcpy(a, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, M * M * 8);
  cudaFuncSetAttribute(kern<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, M * M * 8);
  kern<1><<<1, 512, M * M * 8>>>(a, t, o1); cudaDeviceSynchronize(); long long c1 = *t;
  kern<2><<<1, 512, M * M * 8>>>(a, t, o2); cudaDeviceSynchronize(); long long c2 = *t;
  cudaFuncSetAttribute(kern<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, M * M * 8);
  double* o3; cudaMalloc(&o3, 8192);
  kern<3><<<1, 512, M * M * 8>>>(a, t, o3); cudaDeviceSynchronize(); long long c3 = *t;
  double r3[1024]; cudaMemcpy(r3, o3, 8192, cudaMemcpyDeviceToHost);
  double r1[1024], r2[1024]; cudaMemcpy(r1, o1, 8192, cudaMemcpyDeviceToHost); cudaMemcpy(r2, o2, 8192, cudaMemcpyDeviceToHost);
  double md = 0; for (int e = 0; e < 1024; ++e) { int i = e % 32, j = e / 32; if (i >= j) { double d = r1[e] - r2[e]; md = fmax(md, fabs(d)); } }
  double md3 = 0; for (int e = 0; e < 1024; ++e) { int i = e % 32, j = e / 32; if (i >= j) md3 = fmax(md3, fabs(r1[e] - r3[e])); }
  printf("batched smem %lld cycles, max|diff| vs smem %.3e\n", c3, md3);
  printf("cycles per 32x32 factorisation (incl. restore): smem %lld  reg %lld  max|diff| %.3e  %s\n", c1, c2, md,
         cudaGetErrorString(cudaGetLastError()));
}
