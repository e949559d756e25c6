// Single-CTA shared-memory Cholesky timing (M = 100): which formulation is fast on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ bool chol_left(double* L, int m, int* s_flag) {
  if (threadIdx.x == 0) *s_flag = 1;
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    for (int i = j + threadIdx.x; i < m; i += blockDim.x) {
      double s = L[i + j * m];
      for (int k = 0; k < j; ++k) s -= L[i + k * m] * L[j + k * m];
      L[i + j * m] = s;
    }
    __syncthreads();
    const double d = L[j + j * m];
    if (!(d > 0.0)) return false;
    const double ljj = sqrt(d), inv = 1.0 / ljj;
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) L[i + j * m] *= inv;
    __syncthreads();
    if (threadIdx.x == 0) L[j + j * m] = ljj;
  }
  __syncthreads();
  return true;
}
__global__ void k1(const double* a, int m, long long* t, double* out) {
  extern __shared__ double sm[];
  __shared__ int flag;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) sm[e] = a[e];
  __syncthreads();
  long long t0 = clock64();
  bool ok = chol_left(sm, m, &flag);
  long long t1 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = ok; }
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) out[e] = sm[e];
}
int main() {
  const int m = 100;
  double* h = new double[m * m];
  for (int i = 0; i < m; ++i) for (int j = 0; j < m; ++j) h[i + j * m] = (i == j ? m : 0.0) + 1.0 / (1 + i + j);
  double *a, *o; long long* t; cudaMalloc(&a, 8 * m * m); cudaMalloc(&o, 8 * m * m); cudaMalloc(&t, 16);
  cudaMemcpy(a, h, 8 * m * m, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int th : {128, 256, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      k1<<<1, th, 8 * m * m>>>(a, m, t, o);
      long long ht[2]; cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
      printf("threads %d: %lld cycles ok %lld (%s)\n", th, ht[0], ht[1], cudaGetErrorString(cudaGetLastError()));
    }
  }
}
